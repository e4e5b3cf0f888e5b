// jm_runtime.cpp — libjitmat: the C ABI (include/jit_mat.h) and the
// specialization runtime behind it.
//
// The paper's runtime (§4; Algorithm 1, 308-349) looks
// up a program-global instantiation cache (line 306, "a DenseMap ... protected
// by a mutex"; Algorithm 1 lines 319 and 347) and on a miss instantiates the
// template from embedded compiler state, optimizes it and JITs it; for CUDA it
// picks the device compiler state by compute capability and emits PTX that the
// driver turns into a fatbin (lines 353-354).  Here:
//   * the cache is a direct-indexed table of slots [kind][addend][dtype][N],
//     published with release/acquire atomics; a hit is one acquire load (no
//     lock), a miss takes the slot's own mutex, so distinct keys compile in
//     parallel and concurrent callers of one key wait for a single compile;
//   * the "embedded compiler state" is the kernel template source, embedded in
//     this library at build time; NVRTC instantiates the name expression
//     "jm::k_update<N, T, jm::Addend::X, jm::Tile::Y>" straight to an sm_100a
//     CUBIN (no PTX JIT, no fatbin), with no include paths (no file access at
//     JIT time);
//   * the CUDA driver API is reached through dlopen("libcuda.so.1"), so the
//     library loads (and its symbols can be checked) on a machine without a
//     GPU; NVRTC is statically linked.
#include "jit_mat.h"

#include <cuda.h>
#include <dlfcn.h>
#include <nvrtc.h>
#include <nvtx3/nvToolsExt.h>   // header-only NVTX3: no-ops unless a profiler injects itself

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <type_traits>
#include <vector>

#include "../kernels/jm_plan.h"

extern "C" {
extern const unsigned char jm_embedded_kernel_src[];
extern const char jm_build_digest[];   // sha256 hex of the build inputs (_build.py)
extern const unsigned long long jm_embedded_kernel_src_len;
extern const unsigned char jm_embedded_aot_cubin[];
extern const unsigned long long jm_embedded_aot_cubin_len;
}

namespace {

// ------------------------------------------------------------------ errors
thread_local std::string t_err;

int fail(int code, const char *fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  t_err = buf;
  return code;
}

// ------------------------------------------------------------------ driver API
struct Driver {
  void *handle = nullptr;
  decltype(&cuInit) Init = nullptr;
  decltype(&cuDeviceGet) DeviceGet = nullptr;
  decltype(&cuDeviceGetAttribute) DeviceGetAttribute = nullptr;
  decltype(&cuDevicePrimaryCtxRetain) PrimaryCtxRetain = nullptr;
  decltype(&cuDevicePrimaryCtxRelease) PrimaryCtxRelease = nullptr;
  decltype(&cuCtxGetCurrent) CtxGetCurrent = nullptr;
  decltype(&cuCtxSetCurrent) CtxSetCurrent = nullptr;
  decltype(&cuCtxGetDevice) CtxGetDevice = nullptr;
  decltype(&cuModuleLoadData) ModuleLoadData = nullptr;
  decltype(&cuModuleUnload) ModuleUnload = nullptr;
  decltype(&cuModuleGetFunction) ModuleGetFunction = nullptr;
  decltype(&cuFuncGetAttribute) FuncGetAttribute = nullptr;
  decltype(&cuFuncSetAttribute) FuncSetAttribute = nullptr;
  decltype(&cuLaunchKernel) LaunchKernel = nullptr;
  decltype(&cuStreamSynchronize) StreamSynchronize = nullptr;
  decltype(&cuStreamCreate) StreamCreate = nullptr;
  decltype(&cuStreamDestroy) StreamDestroy = nullptr;
  decltype(&cuStreamWaitEvent) StreamWaitEvent = nullptr;
  decltype(&cuEventCreate) EventCreate = nullptr;
  decltype(&cuEventDestroy) EventDestroy = nullptr;
  decltype(&cuEventRecord) EventRecord = nullptr;
  decltype(&cuMemAlloc) MemAlloc = nullptr;
  decltype(&cuMemFree) MemFree = nullptr;
  decltype(&cuMemcpyHtoDAsync) MemcpyHtoDAsync = nullptr;
  decltype(&cuMemcpyDtoHAsync) MemcpyDtoHAsync = nullptr;
  decltype(&cuMemsetD8Async) MemsetD8Async = nullptr;
  decltype(&cuGetErrorString) GetErrorString = nullptr;
  decltype(&cuOccupancyMaxActiveBlocksPerMultiprocessor) OccupancyMaxActiveBlocks = nullptr;
  decltype(&cuPointerGetAttribute) PointerGetAttribute = nullptr;
};

Driver D;
std::mutex g_driver_mu;

typedef CUresult (*GetProcFn)(const char *, void **, int, cuuint64_t, CUdriverProcAddressQueryResult *);

int load_driver() {
  std::lock_guard<std::mutex> lk(g_driver_mu);
  if (D.handle) return JM_OK;
  void *h = dlopen("libcuda.so.1", RTLD_NOW | RTLD_LOCAL);
  if (!h) return fail(JM_E_CUDA, "CUDA driver libcuda.so.1 not found: %s", dlerror());
  GetProcFn gp = (GetProcFn)dlsym(h, "cuGetProcAddress_v2");
  if (!gp) return fail(JM_E_CUDA, "driver lacks cuGetProcAddress_v2 (driver too old for CUDA 12)");
  bool ok = true;
  auto get = [&](const char *name, auto &fp) {
    void *p = nullptr;
    CUdriverProcAddressQueryResult st;
    CUresult r = gp(name, &p, CUDA_VERSION, CU_GET_PROC_ADDRESS_DEFAULT, &st);
    if (r != CUDA_SUCCESS || !p) ok = false;
    fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(p);
  };
  get("cuInit", D.Init);
  get("cuDeviceGet", D.DeviceGet);
  get("cuDeviceGetAttribute", D.DeviceGetAttribute);
  get("cuDevicePrimaryCtxRetain", D.PrimaryCtxRetain);
  get("cuDevicePrimaryCtxRelease", D.PrimaryCtxRelease);
  get("cuCtxGetCurrent", D.CtxGetCurrent);
  get("cuCtxSetCurrent", D.CtxSetCurrent);
  get("cuCtxGetDevice", D.CtxGetDevice);
  get("cuModuleLoadData", D.ModuleLoadData);
  get("cuModuleUnload", D.ModuleUnload);
  get("cuModuleGetFunction", D.ModuleGetFunction);
  get("cuFuncGetAttribute", D.FuncGetAttribute);
  get("cuFuncSetAttribute", D.FuncSetAttribute);
  get("cuLaunchKernel", D.LaunchKernel);
  get("cuStreamSynchronize", D.StreamSynchronize);
  get("cuStreamCreate", D.StreamCreate);
  get("cuStreamDestroy", D.StreamDestroy);
  get("cuStreamWaitEvent", D.StreamWaitEvent);
  get("cuEventCreate", D.EventCreate);
  get("cuEventDestroy", D.EventDestroy);
  get("cuEventRecord", D.EventRecord);
  get("cuMemAlloc", D.MemAlloc);
  get("cuMemFree", D.MemFree);
  get("cuMemcpyHtoDAsync", D.MemcpyHtoDAsync);
  get("cuMemcpyDtoHAsync", D.MemcpyDtoHAsync);
  get("cuMemsetD8Async", D.MemsetD8Async);
  get("cuGetErrorString", D.GetErrorString);
  get("cuOccupancyMaxActiveBlocksPerMultiprocessor", D.OccupancyMaxActiveBlocks);
  get("cuPointerGetAttribute", D.PointerGetAttribute);
  if (!ok) {
    dlclose(h);
    return fail(JM_E_CUDA, "could not resolve the CUDA driver entry points");
  }
  D.handle = h;
  return JM_OK;
}

int cu_fail(CUresult r, const char *what) {
  const char *s = nullptr;
  if (D.GetErrorString) D.GetErrorString(r, &s);
  return fail(JM_E_CUDA, "%s: CUDA error %d (%s)", what, (int)r, s ? s : "?");
}
#define CU_TRY(expr, what)                      \
  do {                                          \
    CUresult _r = (expr);                       \
    if (_r != CUDA_SUCCESS) return cu_fail(_r, what); \
  } while (0)

// ------------------------------------------------------------------ cache
enum SlotState { S_EMPTY = 0, S_COMPILING = 1, S_READY = 2, S_FAILED = 3 };

struct Slot {
  std::atomic<int> state{S_EMPTY};
  std::mutex mu;
  CUmodule mod = nullptr;     // owned (specialized kind only)
  CUfunction fn = nullptr;
  jm::Plan plan{};
  int grid_cap = 0;           // SM count x resident CTAs per SM
  int regs = 0, local_bytes = 0;
  long long cubin_bytes = 0;
  double compile_ms = 0.0;
  std::string err;
  std::vector<char> cubin;    // NVRTC output kept for jit_mat_cache_export
  std::string lowered;        // mangled kernel symbol
};

constexpr int NKIND = 3, NADD = 2, NDT = 2, NMAX = JM_N_MAX;
Slot g_slots[NKIND][NADD][NDT][NMAX + 1];
Slot g_mm_slots[2][NDT][NMAX + 1];     // multiply-accumulate: [specialized|generic][dtype][n]
Slot g_mass_slots[2][jm::MASS_MAX + 1][jm::MASS_MAX + 1];   // Laghos mass action: [kind][D][Q]
// the streaming (low-repeat) variant of the specialized update: [addend][dtype][n]
Slot g_stream_slots[NADD][NDT][NMAX + 1];
// the latency variant (a warp per matrix, tiny batches; n*n <= 32): [addend][dtype][n]
constexpr int NLAT = 5;
Slot g_lat_slots[NADD][NDT][NLAT + 1];

struct State {
  std::mutex mu;
  std::atomic<bool> inited{false};
  CUdevice dev = 0;
  int ordinal = -1;
  CUcontext ctx = nullptr;
  int sms = 0, cc_major = 0, cc_minor = 0;
  CUmodule aot = nullptr;
  CUfunction generic[NDT][NADD] = {};
  CUfunction fill[NDT] = {};
  CUfunction checksum[NDT] = {};
  CUdeviceptr sum_buf = 0;    // u64 + f64 for checksum
  std::atomic<void *> stream{nullptr};
  // host-buffer staging (run_host)
  std::mutex host_mu;
  CUdeviceptr hbuf[3] = {0, 0, 0};
  size_t hbuf_bytes = 0;
  CUstream hs[3] = {nullptr, nullptr, nullptr};  // h2d, compute, d2h
  CUevent ev_h2d[3] = {}, ev_cmp[3] = {}, ev_d2h[3] = {};
};
State G;

std::atomic<long long> c_compilations{0}, c_hits{0}, c_misses{0}, c_launches{0}, c_imports{0};
std::atomic<long long> c_programs{0};   // NVRTC programs of the batched compile (JM_FLAG_BATCH_COMPILE)
std::atomic<long long> c_compile_us{0};

bool env_flag(const char *name) {
  const char *v = getenv(name);
  return v && *v && strcmp(v, "0") != 0;
}

int ensure_ctx() {
  CUcontext cur = nullptr;
  CU_TRY(D.CtxGetCurrent(&cur), "cuCtxGetCurrent");
  if (cur != G.ctx) CU_TRY(D.CtxSetCurrent(G.ctx), "cuCtxSetCurrent");
  return JM_OK;
}

const char *tile_name(int t) {
  switch ((jm::Tile)t) {
    case jm::Tile::TPM: return "TPM";
    case jm::Tile::Dmma: return "Dmma";
    case jm::Tile::Tpm2: return "Tpm2";
    case jm::Tile::Tpms: return "Tpms";
    case jm::Tile::F32: return "F32";
    case jm::Tile::Rows: return "Rows";
    case jm::Tile::Reg: return "Reg";
    default: return "Generic";
  }
}

std::string name_expression(int n, int dtype, int addend, bool stream = false) {
  char buf[160];
  snprintf(buf, sizeof buf, "jm::%s%s<%d, %s, jm::Addend::%s, jm::Tile::%s>",
           stream ? "k_update_stream" : "k_update",
           jm::use_mb1(n, dtype, stream) ? "_mb1" : jm::use_rc(n, dtype, stream) ? "_rc" : "", n,
           dtype == JM_F64 ? "double" : "float", addend == JM_ADDEND_ONES ? "Ones" : "Identity",
           tile_name((int)jm::tile_for(n, dtype)));
  return buf;
}

std::string lat_name_expression(int n, int dtype, int addend) {
  char buf[96];
  snprintf(buf, sizeof buf, "jm::k_update_lat<%d, %s, jm::Addend::%s>", n, dtype == JM_F64 ? "double" : "float",
           addend == JM_ADDEND_ONES ? "Ones" : "Identity");
  return buf;
}

// the name expression of an update-op slot (resident / streaming / latency)
std::string update_expression(int op, int n, int dtype, int addend);

std::string mm_name_expression(int n, int dtype) {
  char buf[96];
  snprintf(buf, sizeof buf, "jm::k_matmul<%d, %s>", n, dtype == JM_F64 ? "double" : "float");
  return buf;
}

// NVRTC: instantiate name expressions of the embedded template source in ONE
// program -> one sm_100a cubin holding every instantiation (+ the lowered,
// i.e. mangled, symbol of each).  One expression per call is the per-key
// miss path; several are the batched compile of jit_mat_run_many (the
// template source is parsed once for all of them — the paper's "maximal,
// incremental reuse of the state of the compiler").
int nvrtc_compile_exprs(const std::vector<std::string> &exprs, std::vector<char> &cubin,
                        std::vector<std::string> &lowered, std::string &log) {
  const std::string src((const char *)jm_embedded_kernel_src, (size_t)jm_embedded_kernel_src_len);
  nvrtcProgram prog;
  nvrtcResult r = nvrtcCreateProgram(&prog, src.c_str(), "jm_update.cu", 0, nullptr, nullptr);
  if (r != NVRTC_SUCCESS) {
    log = nvrtcGetErrorString(r);
    return JM_E_COMPILE;
  }
  for (const std::string &e : exprs) nvrtcAddNameExpression(prog, e.c_str());
  const char *opts[] = {"--gpu-architecture=sm_100a", "-std=c++17", "--fmad=true", "-lineinfo",
                        "--ftz=false", "--prec-div=true", "--prec-sqrt=true"};
  r = nvrtcCompileProgram(prog, (int)(sizeof opts / sizeof opts[0]), opts);
  size_t lsz = 0;
  nvrtcGetProgramLogSize(prog, &lsz);
  if (lsz > 1) {
    log.resize(lsz);
    nvrtcGetProgramLog(prog, &log[0]);
  }
  if (r != NVRTC_SUCCESS) {
    log = std::string("NVRTC failed for ") + exprs[0] + (exprs.size() > 1 ? " (+ others)" : "") + ": " +
          nvrtcGetErrorString(r) + "\n" + log;
    nvrtcDestroyProgram(&prog);
    return JM_E_COMPILE;
  }
  lowered.clear();
  for (const std::string &e : exprs) {
    const char *low = nullptr;
    nvrtcGetLoweredName(prog, e.c_str(), &low);
    lowered.emplace_back(low ? low : "");
  }
  size_t csz = 0;
  nvrtcGetCUBINSize(prog, &csz);
  cubin.resize(csz);
  nvrtcGetCUBIN(prog, cubin.data());
  nvrtcDestroyProgram(&prog);
  if (const char *dir = getenv("JIT_MAT_DUMP_CUBIN")) {   // inspection hook: cuobjdump -sass the real cubin
    std::string fn = std::string(dir) + "/" + lowered[0] + (exprs.size() > 1 ? ".multi" : "") + ".cubin";
    if (FILE *f = fopen(fn.c_str(), "wb")) {
      fwrite(cubin.data(), 1, cubin.size(), f);
      fclose(f);
    }
  }
  return JM_OK;
}

int nvrtc_compile_expr(const std::string &expr, std::vector<char> &cubin, std::string &lowered,
                       std::string &log) {
  std::vector<std::string> low;
  const int rc = nvrtc_compile_exprs({expr}, cubin, low, log);
  if (rc == JM_OK) lowered = low[0];
  return rc;
}

int finish_function(Slot &s, CUfunction fn) {
  int v = 0;
  D.FuncGetAttribute(&v, CU_FUNC_ATTRIBUTE_NUM_REGS, fn);
  s.regs = v;
  D.FuncGetAttribute(&v, CU_FUNC_ATTRIBUTE_LOCAL_SIZE_BYTES, fn);
  s.local_bytes = v;
  // A failure here is a property of the compiled kernel and its plan on this
  // device (shared memory above the limit, no CTA fits), not a transient driver
  // state: JM_E_COMPILE, so the slot is marked FAILED and not recompiled per call.
  CUresult cr = CUDA_SUCCESS;
  if (s.plan.smem > 48 * 1024 &&
      (cr = D.FuncSetAttribute(fn, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, s.plan.smem)) != CUDA_SUCCESS) {
    cu_fail(cr, "cuFuncSetAttribute(max dynamic smem)");
    return fail(JM_E_COMPILE, "plan needs %d B of shared memory: %s", s.plan.smem, t_err.c_str());
  }
  int nb = 0;
  if ((cr = D.OccupancyMaxActiveBlocks(&nb, fn, s.plan.threads, (size_t)s.plan.smem)) != CUDA_SUCCESS) {
    cu_fail(cr, "cuOccupancyMaxActiveBlocksPerMultiprocessor");
    return fail(JM_E_COMPILE, "%s", t_err.c_str());
  }
  if (nb < 1) return fail(JM_E_COMPILE, "kernel cannot be resident (threads %d, smem %d)", s.plan.threads, s.plan.smem);
  s.grid_cap = nb * G.sms;
  s.fn = fn;
  return JM_OK;
}

// ops: the Eigen-benchmark update (k_update) and the batched multiply-accumulate
// of the RAJA benchmark (k_matmul, Listing 8)
// and the streaming variant of k_update (k_update_stream, jm::plan_stream)
enum { OP_UPDATE = 0, OP_MATMUL = 1, OP_MASS = 2, OP_UPDATE_STREAM = 3, OP_UPDATE_LAT = 4 };

// (for OP_MASS: n = D = NUM_DOFS_1D, extra = Q = NUM_QUAD_1D)
jm::Plan plan_for(int op, int n, int dtype, int extra) {
  return op == OP_MATMUL          ? jm::plan_matmul(n, dtype)
         : op == OP_MASS          ? jm::plan_mass(n, extra)
         : op == OP_UPDATE_STREAM ? jm::plan_stream(n, dtype)
         : op == OP_UPDATE_LAT    ? jm::plan_lat(n, dtype)
                                  : jm::plan_specialized(n, dtype);
}

std::string update_expression(int op, int n, int dtype, int addend) {
  return op == OP_UPDATE_LAT ? lat_name_expression(n, dtype, addend)
                             : name_expression(n, dtype, addend, op == OP_UPDATE_STREAM);
}

std::string mass_name_expression(int d, int q) {
  char buf[64];
  snprintf(buf, sizeof buf, "jm::k_mass<%d, %d>", d, q);
  return buf;
}

// Load a specialized cubin into a slot (after NVRTC, or from an imported blob).
int install_cubin(Slot &s, int op, int n, int dtype, int extra, std::vector<char> &&cubin,
                  const std::string &lowered) {
  int rc = ensure_ctx();
  if (rc != JM_OK) return rc;
  CUmodule mod = nullptr;
  CUresult cr = D.ModuleLoadData(&mod, cubin.data());
  if (cr != CUDA_SUCCESS) {
    cu_fail(cr, "cuModuleLoadData(NVRTC cubin)");
    s.err = t_err;
    return JM_E_COMPILE;
  }
  CUfunction fn = nullptr;
  cr = D.ModuleGetFunction(&fn, mod, lowered.c_str());
  if (cr != CUDA_SUCCESS) {
    D.ModuleUnload(mod);
    cu_fail(cr, "cuModuleGetFunction");
    s.err = t_err;
    return JM_E_COMPILE;
  }
  s.plan = plan_for(op, n, dtype, extra);
  s.mod = mod;
  s.cubin_bytes = (long long)cubin.size();
  rc = finish_function(s, fn);
  if (rc != JM_OK) {
    D.ModuleUnload(mod);
    s.mod = nullptr;
    s.err = t_err;
    return rc;
  }
  s.cubin = std::move(cubin);
  s.lowered = lowered;
  return JM_OK;
}

// NVTX range for the duration of a scope (jm:compile / jm:run,
// for ncu --nvtx filtering and timeline tools)
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

int compile_slot(Slot &s, int op, int n, int dtype, int addend) {
  NvtxRange nvtx("jm:compile");
  const auto t0 = std::chrono::steady_clock::now();
  c_compilations++;
  std::vector<char> cubin;
  std::string lowered, log;
  const std::string expr = op == OP_MATMUL ? mm_name_expression(n, dtype)
                           : op == OP_MASS ? mass_name_expression(n, addend)
                                           : update_expression(op, n, dtype, addend);
  int rc = nvrtc_compile_expr(expr, cubin, lowered, log);
  if (rc != JM_OK) {
    s.err = log;
    return fail(rc, "%s", log.c_str());
  }
  if ((rc = install_cubin(s, op, n, dtype, addend, std::move(cubin), lowered)) != JM_OK) return rc;
  const double ms =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  s.compile_ms = ms;
  c_compile_us += (long long)(ms * 1000.0);
  if (env_flag("JIT_MAT_LOG"))
    fprintf(stderr, "[jitmat] compiled %s in %.1f ms (%lld B cubin, %d regs, %d B local)\n",
            expr.c_str(), ms, s.cubin_bytes, s.regs, s.local_bytes);
  return JM_OK;
}

int check_key(int n, int dtype, int addend, int kind) {
  if (n <= 0) return fail(JM_E_INVALID, "n must be >= 1 (got %d)", n);
  if (n > JM_N_MAX) return fail(JM_E_UNSUPPORTED, "n = %d exceeds the supported maximum %d", n, JM_N_MAX);
  if (dtype != JM_F32 && dtype != JM_F64) return fail(JM_E_UNSUPPORTED, "dtype %d not supported (f32/f64 only)", dtype);
  if (addend != JM_ADDEND_ONES && addend != JM_ADDEND_IDENTITY) return fail(JM_E_INVALID, "addend %d invalid", addend);
  if (kind != JM_KIND_SPECIALIZED && kind != JM_KIND_GENERIC && kind != JM_KIND_AOT_SPECIALIZED)
    return fail(JM_E_INVALID, "kind %d invalid", kind);
  return JM_OK;
}

int acquire_slot(Slot &s, int op, int n, int dtype, int addend, int kind, Slot **out);

// Algorithm 1 (PAPER.md:319 lookup, :347 store) with per-key once semantics.
int lookup_op(int op, int n, int dtype, int addend, int kind, Slot **out) {
  int rc = check_key(n, dtype, addend, kind);
  if (rc != JM_OK) return rc;
  if (!G.inited.load(std::memory_order_acquire)) return fail(JM_E_NOT_INITIALIZED, "jit_mat_init has not been called");
  if (op == OP_MATMUL && kind == JM_KIND_AOT_SPECIALIZED)
    return fail(JM_E_UNSUPPORTED, "no ahead-of-time specialization of the multiply-accumulate");
  Slot &s = op == OP_MATMUL ? g_mm_slots[kind][dtype][n] : g_slots[kind][addend][dtype][n];
  return acquire_slot(s, op, n, dtype, addend, kind, out);
}

// The slot state machine of Algorithm 1 (hit: one acquire load; miss: the
// slot's mutex, then compile once).  For OP_MASS, n = D and `addend` = Q.
int acquire_slot(Slot &s, int op, int n, int dtype, int addend, int kind, Slot **out) {
  int rc = JM_OK;
  int st = s.state.load(std::memory_order_acquire);
  if (st == S_READY) {
    c_hits++;
    *out = &s;
    return JM_OK;
  }
  if (st == S_FAILED) return fail(JM_E_COMPILE, "%s", s.err.c_str());
  c_misses++;
  std::lock_guard<std::mutex> lk(s.mu);
  st = s.state.load(std::memory_order_acquire);
  if (st == S_READY) { *out = &s; return JM_OK; }
  if (st == S_FAILED) return fail(JM_E_COMPILE, "%s", s.err.c_str());
  if (kind == JM_KIND_GENERIC) return fail(JM_E_INVALID, "generic slot not seeded");
  if (kind == JM_KIND_AOT_SPECIALIZED)
    return fail(JM_E_UNSUPPORTED, "no ahead-of-time specialization for n=%d %s (available: n = 3, 7, 16, double)",
                n, dtype == JM_F64 ? "double" : "float");
  s.state.store(S_COMPILING, std::memory_order_relaxed);
  rc = compile_slot(s, op, n, dtype, addend);
  if (rc != JM_OK) {
    if (rc == JM_E_COMPILE) {
      s.state.store(S_FAILED, std::memory_order_release);
    } else {
      s.state.store(S_EMPTY, std::memory_order_release);   // transient (driver) error: retry later
    }
    return rc;
  }
  s.state.store(S_READY, std::memory_order_release);
  *out = &s;
  return JM_OK;
}

int lookup(int n, int dtype, int addend, int kind, Slot **out) {
  return lookup_op(OP_UPDATE, n, dtype, addend, kind, out);
}

// Resident or streaming kernel for this call?  The roofline decides
// (jm_plan.h, plan_stream): stream when repeat * (n + 1) is below the switch
// point, i.e. when the call is bound by moving each matrix in and out once.
// JIT_MAT_STREAM=0 / =1 force the resident / streaming kernel (where the
// tiling kind has one); JIT_MAT_STREAM_RN moves the switch point.
int stream_rn(int n, int dtype) {
  static const int rn = [] {
    const char *e = getenv("JIT_MAT_STREAM_RN");
    return e && *e ? atoi(e) : -1;
  }();
  return rn >= 0 ? rn : jm::stream_rn(n, dtype);
}
bool want_stream(int n, int dtype, int kind, int64_t repeat, unsigned flags = 0) {
  if (kind != JM_KIND_SPECIALIZED || !jm::stream_ok(n, dtype)) return false;
  if (flags & JM_FLAG_RESIDENT) return false;
  if (flags & JM_FLAG_STREAMING) return true;
  static const int force = [] {
    const char *e = getenv("JIT_MAT_STREAM");
    return e && *e ? atoi(e) : -1;
  }();
  if (force >= 0) return force > 0;
  const int64_t rn = repeat * (int64_t)(n + 1);
  return rn < (int64_t)stream_rn(n, dtype) && rn >= (int64_t)jm::stream_lo(n, dtype);
}

// The latency variant: a warp per matrix for tiny batches (every matrix gets
// its own warp: batch <= LAT_BATCH_PER_SM x SMs), n*n <= 32, or forced by
// JM_FLAG_LATENCY; JM_FLAG_RESIDENT / JM_FLAG_STREAMING and
// JIT_MAT_LATENCY=0 keep it off.
bool want_lat(int n, int dtype, int kind, int64_t batch, unsigned flags) {
  (void)dtype;
  if (kind != JM_KIND_SPECIALIZED || !jm::lat_ok(n)) return false;
  if (flags & JM_FLAG_LATENCY) return true;
  if (flags & (JM_FLAG_RESIDENT | JM_FLAG_STREAMING)) return false;
  static const bool off = [] {
    const char *e = getenv("JIT_MAT_LATENCY");
    return e && *e && strcmp(e, "0") == 0;
  }();
  return !off && batch > 0 && batch <= (int64_t)jm::LAT_BATCH_PER_SM * G.sms;
}

// variant of a run: 0 resident, 1 streaming, 2 latency
int variant_of(const jm_run_desc &d) {
  if (want_lat(d.n, d.dtype, d.kind, d.batch, d.flags)) return 2;
  return want_stream(d.n, d.dtype, d.kind, d.repeat, d.flags) ? 1 : 0;
}

Slot &slot_of(int n, int dtype, int addend, int kind, int variant) {
  return variant == 2 ? g_lat_slots[addend][dtype][n]
         : variant == 1 ? g_stream_slots[addend][dtype][n] : g_slots[kind][addend][dtype][n];
}

int op_of_variant(int variant) { return variant == 2 ? OP_UPDATE_LAT : variant == 1 ? OP_UPDATE_STREAM : OP_UPDATE; }

// the kernel a run descriptor launches (key checked by the caller)
int lookup_run(const jm_run_desc &d, Slot **out) {
  const int v = variant_of(d);
  if (v == 0) return lookup(d.n, d.dtype, d.addend, d.kind, out);
  if (!G.inited.load(std::memory_order_acquire)) return fail(JM_E_NOT_INITIALIZED, "jit_mat_init has not been called");
  return acquire_slot(slot_of(d.n, d.dtype, d.addend, JM_KIND_SPECIALIZED, v), op_of_variant(v), d.n, d.dtype,
                      d.addend, JM_KIND_SPECIALIZED, out);
}

int launch(Slot &s, int n, int64_t batch, int64_t repeat, const void *in, void *out, CUstream stream,
           int kind) {
  const long long mpc = s.plan.mpc;
  const long long nchunks = (batch + mpc - 1) / mpc;
  const unsigned grid = (unsigned)(nchunks < s.grid_cap ? nchunks : s.grid_cap);
  long long b = batch;
  int r = (int)repeat;
  CUdeviceptr pin = (CUdeviceptr)in, pout = (CUdeviceptr)out;
  void *args_spec[] = {&pin, &pout, &b, &r};
  int nn = n;
  void *args_gen[] = {&pin, &pout, &b, &r, &nn};
  CU_TRY(D.LaunchKernel(s.fn, grid, 1, 1, (unsigned)s.plan.threads, 1, 1, (unsigned)s.plan.smem, stream,
                        kind == JM_KIND_GENERIC ? args_gen : args_spec, nullptr),
         "cuLaunchKernel(update)");
  c_launches++;
  return JM_OK;
}

int validate_run(const jm_run_desc *d) {
  if (!d) return fail(JM_E_INVALID, "NULL descriptor");
  int rc = check_key(d->n, d->dtype, d->addend, d->kind);
  if (rc != JM_OK) return rc;
  if (d->batch < 0) return fail(JM_E_INVALID, "batch must be >= 0 (got %lld)", (long long)d->batch);
  if (d->repeat < 0 || d->repeat > JM_REPEAT_MAX)
    return fail(JM_E_INVALID, "repeat must be in [0, 2^31) (got %lld)", (long long)d->repeat);
  if (!G.inited.load(std::memory_order_acquire)) return fail(JM_E_NOT_INITIALIZED, "jit_mat_init has not been called");
  if (d->batch == 0) return JM_OK;
  if (!d->in || !d->out) return fail(JM_E_INVALID, "NULL buffer");
  const size_t es = d->dtype == JM_F64 ? 8 : 4;
  const unsigned long long bytes = (unsigned long long)d->batch * d->n * d->n * es;
  const unsigned long long a = (unsigned long long)d->in, b = (unsigned long long)d->out;
  if (a != b && a < b + bytes && b < a + bytes)
    return fail(JM_E_INVALID, "in and out partially overlap (only exact aliasing is allowed)");
  if (!(d->flags & JM_FLAG_HOST_BUFFERS) && ((a | b) & 15))
    return fail(JM_E_ALIGN, "in/out must be 16-byte aligned");
  return JM_OK;
}

int sync_if(unsigned flags, CUstream st) {
  if ((flags & JM_FLAG_SYNC) || env_flag("JIT_MAT_SYNC")) CU_TRY(D.StreamSynchronize(st), "kernel execution");
  return JM_OK;
}

// Host buffers: stream chunks H2D -> update in place on the device -> D2H,
// three library-owned device buffers in rotation on three streams so the two
// copy directions and the kernel overlap.
int run_host(const jm_run_desc *d, Slot &s) {
  std::lock_guard<std::mutex> lk(G.host_mu);
  const size_t es = d->dtype == JM_F64 ? 8 : 4;
  const size_t mb = (size_t)d->n * d->n * es;
  size_t chunk_bytes = (size_t)64 << 20;
  if (const char *e = getenv("JIT_MAT_HOST_CHUNK_MB")) chunk_bytes = (size_t)atoll(e) << 20;
  long long per = (long long)(chunk_bytes / mb);
  per -= per % 4;                        // keep chunk starts 16-B aligned
  if (per < 4) per = 4;
  const size_t need = (size_t)per * mb;
  if (G.hbuf_bytes < need) {
    for (int i = 0; i < 3; ++i)
      if (G.hbuf[i]) { D.MemFree(G.hbuf[i]); G.hbuf[i] = 0; }
    G.hbuf_bytes = 0;
    for (int i = 0; i < 3; ++i) CU_TRY(D.MemAlloc(&G.hbuf[i], need), "cuMemAlloc(host staging)");
    G.hbuf_bytes = need;
  }
  if (!G.hs[0]) {
    for (int i = 0; i < 3; ++i) {
      CU_TRY(D.StreamCreate(&G.hs[i], CU_STREAM_NON_BLOCKING), "cuStreamCreate");
      CU_TRY(D.EventCreate(&G.ev_h2d[i], CU_EVENT_DISABLE_TIMING), "cuEventCreate");
      CU_TRY(D.EventCreate(&G.ev_cmp[i], CU_EVENT_DISABLE_TIMING), "cuEventCreate");
      CU_TRY(D.EventCreate(&G.ev_d2h[i], CU_EVENT_DISABLE_TIMING), "cuEventCreate");
    }
  }
  const char *hin = (const char *)d->in;
  char *hout = (char *)d->out;
  long long c = 0;
  for (long long b0 = 0; b0 < d->batch; b0 += per, ++c) {
    const long long cnt = (d->batch - b0) < per ? (d->batch - b0) : per;
    const size_t bytes = (size_t)cnt * mb;
    const int k = (int)(c % 3);
    if (c >= 3) CU_TRY(D.StreamWaitEvent(G.hs[0], G.ev_d2h[k], 0), "cuStreamWaitEvent");
    CU_TRY(D.MemcpyHtoDAsync(G.hbuf[k], hin + (size_t)b0 * mb, bytes, G.hs[0]), "cuMemcpyHtoDAsync");
    CU_TRY(D.EventRecord(G.ev_h2d[k], G.hs[0]), "cuEventRecord");
    CU_TRY(D.StreamWaitEvent(G.hs[1], G.ev_h2d[k], 0), "cuStreamWaitEvent");
    int rc = launch(s, d->n, cnt, d->repeat, (const void *)G.hbuf[k], (void *)G.hbuf[k], G.hs[1], d->kind);
    if (rc != JM_OK) return rc;
    CU_TRY(D.EventRecord(G.ev_cmp[k], G.hs[1]), "cuEventRecord");
    CU_TRY(D.StreamWaitEvent(G.hs[2], G.ev_cmp[k], 0), "cuStreamWaitEvent");
    CU_TRY(D.MemcpyDtoHAsync(hout + (size_t)b0 * mb, G.hbuf[k], bytes, G.hs[2]), "cuMemcpyDtoHAsync");
    CU_TRY(D.EventRecord(G.ev_d2h[k], G.hs[2]), "cuEventRecord");
  }
  CU_TRY(D.StreamSynchronize(G.hs[2]), "host-buffer pipeline");
  CU_TRY(D.StreamSynchronize(G.hs[1]), "host-buffer pipeline");
  return JM_OK;
}

int run_impl(const jm_run_desc *d) {
  NvtxRange nvtx("jm:run");
  int rc = validate_run(d);
  if (rc != JM_OK || d->batch == 0) return rc;
  Slot *s = nullptr;
  if ((rc = lookup_run(*d, &s)) != JM_OK) return rc;
  if ((rc = ensure_ctx()) != JM_OK) return rc;
  if (d->flags & JM_FLAG_HOST_BUFFERS) return run_host(d, *s);
  CUstream st = (CUstream)(d->stream ? d->stream : G.stream.load(std::memory_order_relaxed));
  if ((rc = launch(*s, d->n, d->batch, d->repeat, d->in, d->out, st, d->kind)) != JM_OK) return rc;
  return sync_if(d->flags, st);
}

// Batched specialization (jit_mat_run_many with JM_FLAG_BATCH_COMPILE): the
// distinct cold specialized keys of the descriptors are split into G groups
// (G = JIT_MAT_COMPILE_GROUPS, default the hardware threads, at most the key
// count), each group is ONE NVRTC program with one name expression per key,
// and the groups compile on G host threads.  The resulting cubin (all of a
// group's kernels) is then loaded into each key's slot under that slot's own
// lock; a slot another thread made READY meanwhile is left alone, so there
// is no lock ordering to get wrong (at worst a key is compiled twice).
struct ColdKey {
  int op, n, dtype, addend;
  Slot *slot;
};
int batch_compile(const jm_run_desc *d, const std::vector<int> &todo) {
  std::vector<ColdKey> keys;
  for (int i : todo) {
    const int v = variant_of(d[i]);
    if (d[i].kind != JM_KIND_SPECIALIZED) continue;   // generic / AoT slots are seeded, never compiled
    Slot *s = &slot_of(d[i].n, d[i].dtype, d[i].addend, d[i].kind, v);
    bool dup = false;
    for (const ColdKey &k : keys) dup |= (k.slot == s);
    if (!dup) keys.push_back({op_of_variant(v), d[i].n, d[i].dtype, d[i].addend, s});
  }
  if (keys.empty()) return JM_OK;
  int groups = (int)std::thread::hardware_concurrency();
  if (const char *e = getenv("JIT_MAT_COMPILE_GROUPS")) groups = atoi(e);
  if (groups < 1) groups = 1;
  if (groups > (int)keys.size()) groups = (int)keys.size();
  // balance the groups by expected compile cost (larger n: bigger kernels)
  std::vector<int> order(keys.size());
  for (size_t i = 0; i < order.size(); ++i) order[i] = (int)i;
  std::sort(order.begin(), order.end(), [&](int a, int b) { return keys[a].n > keys[b].n; });
  std::vector<std::vector<int>> part((size_t)groups);
  std::vector<long long> load((size_t)groups, 0);
  for (int i : order) {
    const size_t g = (size_t)(std::min_element(load.begin(), load.end()) - load.begin());
    part[g].push_back(i);
    load[g] += 64 + (long long)keys[(size_t)i].n * keys[(size_t)i].n;
  }
  std::vector<int> rcs((size_t)groups, JM_OK);
  std::vector<std::string> errs((size_t)groups);
  std::vector<std::thread> th;
  for (int g = 0; g < groups; ++g)
    th.emplace_back([&, g] {
      NvtxRange nvtx("jm:compile");
      const auto t0 = std::chrono::steady_clock::now();
      std::vector<std::string> exprs, lowered;
      for (int i : part[(size_t)g]) {
        const ColdKey &k = keys[(size_t)i];
        exprs.push_back(update_expression(k.op, k.n, k.dtype, k.addend));
      }
      std::vector<char> cubin;
      std::string log;
      int rc = nvrtc_compile_exprs(exprs, cubin, lowered, log);
      if (rc != JM_OK) { rcs[(size_t)g] = rc; errs[(size_t)g] = log; return; }
      const double ms =
          std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
      for (size_t j = 0; j < exprs.size(); ++j) {
        const ColdKey &k = keys[(size_t)part[(size_t)g][j]];
        Slot &s = *k.slot;
        std::lock_guard<std::mutex> lk(s.mu);
        if (s.state.load(std::memory_order_acquire) == S_READY) continue;
        std::vector<char> copy(cubin);
        rc = install_cubin(s, k.op, k.n, k.dtype, k.addend, std::move(copy), lowered[j]);
        if (rc != JM_OK) {
          s.err = t_err;
          if (rc == JM_E_COMPILE) s.state.store(S_FAILED, std::memory_order_release);
          rcs[(size_t)g] = rc;
          errs[(size_t)g] = t_err;
          continue;
        }
        s.compile_ms = ms / (double)exprs.size();   // the program's time, shared by its keys
        c_compilations++;
        c_compile_us += (long long)(s.compile_ms * 1000.0);
        s.state.store(S_READY, std::memory_order_release);
      }
      c_programs++;
    });
  for (auto &t : th) t.join();
  for (int g = 0; g < groups; ++g)
    if (rcs[(size_t)g] != JM_OK) return fail(rcs[(size_t)g], "batched compile: %s", errs[(size_t)g].c_str());
  return JM_OK;
}

// Mixed-N: resolve every key (cold keys compile concurrently), then fork the
// groups over a pool of streams and join them back into the caller's stream.
constexpr int POOL = 8;
std::mutex g_pool_mu;
CUstream g_pool[POOL] = {};
CUevent g_fork = nullptr, g_join[POOL] = {};

int run_many_impl(const jm_run_desc *d, int count, void *stream, unsigned flags) {
  if (count < 0 || (count > 0 && !d)) return fail(JM_E_INVALID, "bad descriptor array");
  for (int i = 0; i < count; ++i) {
    if (d[i].flags & JM_FLAG_HOST_BUFFERS) return fail(JM_E_INVALID, "descriptor %d: host buffers not allowed", i);
    if (d[i].stream) return fail(JM_E_INVALID, "descriptor %d: per-descriptor stream not allowed", i);
    int rc = validate_run(&d[i]);
    if (rc != JM_OK) {
      t_err = "descriptor " + std::to_string(i) + ": " + t_err;
      return rc;
    }
  }
  // 1. specialize: distinct cold keys in parallel (one host thread per key),
  // or (JM_FLAG_BATCH_COMPILE) as a few NVRTC programs of several name
  // expressions each, compiled in parallel
  std::vector<Slot *> slots((size_t)count, nullptr);
  std::vector<int> todo;
  for (int i = 0; i < count; ++i) {
    if (d[i].batch == 0) continue;
    Slot &s = slot_of(d[i].n, d[i].dtype, d[i].addend, d[i].kind, variant_of(d[i]));
    if (s.state.load(std::memory_order_acquire) != S_READY) todo.push_back(i);
  }
  if ((flags & JM_FLAG_BATCH_COMPILE) && todo.size() > 1) {
    int rc = batch_compile(d, todo);
    if (rc != JM_OK) return rc;
  } else if (todo.size() > 1) {
    std::vector<std::thread> th;
    std::vector<int> rcs(todo.size(), JM_OK);
    std::vector<std::string> errs(todo.size());
    for (size_t t = 0; t < todo.size(); ++t)
      th.emplace_back([&, t] {
        Slot *s = nullptr;
        const jm_run_desc &x = d[todo[t]];
        rcs[t] = lookup_run(x, &s);
        if (rcs[t] != JM_OK) errs[t] = t_err;
      });
    for (auto &t : th) t.join();
    for (size_t t = 0; t < todo.size(); ++t)
      if (rcs[t] != JM_OK) return fail(rcs[t], "descriptor %d: %s", todo[t], errs[t].c_str());
  }
  for (int i = 0; i < count; ++i) {
    if (d[i].batch == 0) continue;
    int rc = lookup_run(d[i], &slots[(size_t)i]);
    if (rc != JM_OK) return rc;
  }
  int rc = ensure_ctx();
  if (rc != JM_OK) return rc;
  CUstream st = (CUstream)(stream ? stream : G.stream.load(std::memory_order_relaxed));
  // 2. fork / launch / join; biggest groups first, round-robin over the pool
  std::vector<int> order;
  for (int i = 0; i < count; ++i)
    if (d[i].batch > 0) order.push_back(i);
  auto work = [&](int i) { return (double)d[i].batch * d[i].n * d[i].n * (d[i].n + 1) * (double)(d[i].repeat + 1); };
  std::sort(order.begin(), order.end(), [&](int a, int b) { return work(a) > work(b); });
  std::lock_guard<std::mutex> lk(g_pool_mu);
  if (!g_fork) {
    CU_TRY(D.EventCreate(&g_fork, CU_EVENT_DISABLE_TIMING), "cuEventCreate");
    for (int p = 0; p < POOL; ++p) {
      CU_TRY(D.StreamCreate(&g_pool[p], CU_STREAM_NON_BLOCKING), "cuStreamCreate");
      CU_TRY(D.EventCreate(&g_join[p], CU_EVENT_DISABLE_TIMING), "cuEventCreate");
    }
  }
  const int used = (int)std::min<size_t>(order.size(), POOL);
  if (used == 0) return JM_OK;
  CU_TRY(D.EventRecord(g_fork, st), "cuEventRecord(fork)");
  for (int p = 0; p < used; ++p) CU_TRY(D.StreamWaitEvent(g_pool[p], g_fork, 0), "cuStreamWaitEvent(fork)");
  for (size_t k = 0; k < order.size(); ++k) {
    const jm_run_desc &x = d[order[k]];
    rc = launch(*slots[(size_t)order[k]], x.n, x.batch, x.repeat, x.in, x.out, g_pool[k % used], x.kind);
    if (rc != JM_OK) return rc;
  }
  for (int p = 0; p < used; ++p) {
    CU_TRY(D.EventRecord(g_join[p], g_pool[p]), "cuEventRecord(join)");
    CU_TRY(D.StreamWaitEvent(st, g_join[p], 0), "cuStreamWaitEvent(join)");
  }
  return sync_if(flags, st);
}

void seed_generic_slots() {
  for (int dt = 0; dt < NDT; ++dt)
    for (int ad = 0; ad < NADD; ++ad)
      for (int n = 1; n <= NMAX; ++n) {
        Slot &s = g_slots[JM_KIND_GENERIC][ad][dt][n];
        s.plan = jm::plan_generic(n, dt);
        s.mod = nullptr;
        s.cubin_bytes = (long long)jm_embedded_aot_cubin_len;
        if (finish_function(s, G.generic[dt][ad]) == JM_OK) s.state.store(S_READY, std::memory_order_release);
        else { s.err = t_err; s.state.store(S_FAILED, std::memory_order_release); }
      }
}

// Explicit (ahead-of-time) specializations take precedence over compiling
// (PAPER.md:176): their slots are READY from the start.
int seed_aot_spec_slots() {
  for (int ad = 0; ad < NADD; ++ad)
    for (int n = 1; n <= NMAX; ++n) {
      if (!jm::aot_spec_available(n, JM_F64)) continue;
      char name[96];
      snprintf(name, sizeof name, "jm_aotspec_double_n%d_%s", n, ad == JM_ADDEND_ONES ? "ones" : "identity");
      CUfunction fn = nullptr;
      CU_TRY(D.ModuleGetFunction(&fn, G.aot, name), name);
      Slot &s = g_slots[JM_KIND_AOT_SPECIALIZED][ad][JM_F64][n];
      s.plan = jm::plan_specialized(n, JM_F64);
      s.mod = nullptr;
      s.cubin_bytes = (long long)jm_embedded_aot_cubin_len;
      int rc = finish_function(s, fn);
      if (rc != JM_OK) return rc;
      s.state.store(S_READY, std::memory_order_release);
    }
  return JM_OK;
}

}  // namespace

// ====================================================================== ABI
extern "C" {

int jit_mat_init(int device) {
  std::lock_guard<std::mutex> lk(G.mu);
  if (G.inited.load()) {
    if (device >= 0 && device != G.ordinal)
      return fail(JM_E_INVALID, "already initialised on device %d", G.ordinal);
    return ensure_ctx();
  }
  int rc = load_driver();
  if (rc != JM_OK) return rc;
  CU_TRY(D.Init(0), "cuInit");
  int ord = device;
  if (ord < 0) {
    CUcontext cur = nullptr;
    CUdevice cd = 0;
    ord = 0;
    if (D.CtxGetCurrent(&cur) == CUDA_SUCCESS && cur && D.CtxGetDevice(&cd) == CUDA_SUCCESS) ord = (int)cd;
  }
  CU_TRY(D.DeviceGet(&G.dev, ord), "cuDeviceGet");
  CU_TRY(D.DeviceGetAttribute(&G.cc_major, CU_DEVICE_ATTRIBUTE_COMPUTE_CAPABILITY_MAJOR, G.dev), "cuDeviceGetAttribute");
  CU_TRY(D.DeviceGetAttribute(&G.cc_minor, CU_DEVICE_ATTRIBUTE_COMPUTE_CAPABILITY_MINOR, G.dev), "cuDeviceGetAttribute");
  CU_TRY(D.DeviceGetAttribute(&G.sms, CU_DEVICE_ATTRIBUTE_MULTIPROCESSOR_COUNT, G.dev), "cuDeviceGetAttribute");
  int major = G.cc_major;
  if (const char *e = getenv("JIT_MAT_FAKE_CC_MAJOR")) major = atoi(e);   // tests of the JM_E_ARCH path
  if (major != 10)
    return fail(JM_E_ARCH, "device %d has compute capability %d.%d; this library targets sm_100a (B200) only",
                ord, major, G.cc_minor);
  CU_TRY(D.PrimaryCtxRetain(&G.ctx, G.dev), "cuDevicePrimaryCtxRetain");
  G.ordinal = ord;
  if ((rc = ensure_ctx()) != JM_OK) return rc;
  CU_TRY(D.ModuleLoadData(&G.aot, jm_embedded_aot_cubin), "cuModuleLoadData(AoT cubin)");
  static const char *gnames[NDT][NADD] = {{"jm_generic_f32_ones", "jm_generic_f32_identity"},
                                          {"jm_generic_f64_ones", "jm_generic_f64_identity"}};
  for (int dt = 0; dt < NDT; ++dt)
    for (int ad = 0; ad < NADD; ++ad) CU_TRY(D.ModuleGetFunction(&G.generic[dt][ad], G.aot, gnames[dt][ad]), gnames[dt][ad]);
  CU_TRY(D.ModuleGetFunction(&G.fill[0], G.aot, "jm_fill_f32"), "jm_fill_f32");
  CU_TRY(D.ModuleGetFunction(&G.fill[1], G.aot, "jm_fill_f64"), "jm_fill_f64");
  CU_TRY(D.ModuleGetFunction(&G.checksum[0], G.aot, "jm_checksum_f32"), "jm_checksum_f32");
  CU_TRY(D.ModuleGetFunction(&G.checksum[1], G.aot, "jm_checksum_f64"), "jm_checksum_f64");
  {
    CUfunction mmg[NDT] = {};
    CU_TRY(D.ModuleGetFunction(&mmg[0], G.aot, "jm_mm_generic_f32"), "jm_mm_generic_f32");
    CU_TRY(D.ModuleGetFunction(&mmg[1], G.aot, "jm_mm_generic_f64"), "jm_mm_generic_f64");
    for (int dt = 0; dt < NDT; ++dt)
      for (int n = 1; n <= NMAX; ++n) {
        Slot &s = g_mm_slots[JM_KIND_GENERIC][dt][n];
        s.plan = jm::plan_matmul_generic(n, dt);
        s.cubin_bytes = (long long)jm_embedded_aot_cubin_len;
        if ((rc = finish_function(s, mmg[dt])) != JM_OK) return rc;
        s.state.store(S_READY, std::memory_order_release);
      }
    CUfunction mg = nullptr;
    CU_TRY(D.ModuleGetFunction(&mg, G.aot, "jm_mass_generic"), "jm_mass_generic");
    for (int d = 1; d <= jm::MASS_MAX; ++d)
      for (int q = 1; q <= jm::MASS_MAX; ++q) {
        Slot &s = g_mass_slots[JM_KIND_GENERIC][d][q];
        s.plan = jm::Plan{(int)jm::Tile::Generic, jm::MASS_THREADS, jm::MASS_THREADS,
                          jm::MASS_THREADS * (2 * d * d + q * q) * 8 + q * d * 8, 1};
        s.cubin_bytes = (long long)jm_embedded_aot_cubin_len;
        if ((rc = finish_function(s, mg)) != JM_OK) return rc;
        s.state.store(S_READY, std::memory_order_release);
      }
  }
  CU_TRY(D.MemAlloc(&G.sum_buf, 16), "cuMemAlloc(checksum)");
  seed_generic_slots();
  if ((rc = seed_aot_spec_slots()) != JM_OK) return rc;
  G.inited.store(true, std::memory_order_release);
  return JM_OK;
}

int jit_mat_shutdown(void) {
  std::lock_guard<std::mutex> lk(G.mu);
  if (!G.inited.load()) return fail(JM_E_NOT_INITIALIZED, "not initialised");
  ensure_ctx();
  G.inited.store(false, std::memory_order_release);
  auto reset = [](Slot &s) {
    std::lock_guard<std::mutex> sl(s.mu);
    if (s.mod) D.ModuleUnload(s.mod);
    s.mod = nullptr;
    s.fn = nullptr;
    s.err.clear();
    s.regs = s.local_bytes = 0;
    s.cubin_bytes = 0;
    s.cubin.clear();
    s.cubin.shrink_to_fit();
    s.lowered.clear();
    s.compile_ms = 0;
    s.state.store(S_EMPTY, std::memory_order_release);
  };
  for (int k = 0; k < NKIND; ++k)
    for (int a = 0; a < NADD; ++a)
      for (int t = 0; t < NDT; ++t)
        for (int n = 0; n <= NMAX; ++n) reset(g_slots[k][a][t][n]);
  for (int k = 0; k < 2; ++k)
    for (int t = 0; t < NDT; ++t)
      for (int n = 0; n <= NMAX; ++n) reset(g_mm_slots[k][t][n]);
  for (int k = 0; k < 2; ++k)
    for (int d = 0; d <= jm::MASS_MAX; ++d)
      for (int q = 0; q <= jm::MASS_MAX; ++q) reset(g_mass_slots[k][d][q]);
  for (int a = 0; a < NADD; ++a)
    for (int t = 0; t < NDT; ++t) {
      for (int n = 0; n <= NMAX; ++n) reset(g_stream_slots[a][t][n]);
      for (int n = 0; n <= NLAT; ++n) reset(g_lat_slots[a][t][n]);
    }
  {
    std::lock_guard<std::mutex> hl(G.host_mu);
    for (int i = 0; i < 3; ++i) {
      if (G.hbuf[i]) D.MemFree(G.hbuf[i]);
      G.hbuf[i] = 0;
      if (G.hs[i]) {
        D.StreamDestroy(G.hs[i]);
        D.EventDestroy(G.ev_h2d[i]);
        D.EventDestroy(G.ev_cmp[i]);
        D.EventDestroy(G.ev_d2h[i]);
      }
      G.hs[i] = nullptr;
    }
    G.hbuf_bytes = 0;
  }
  {
    std::lock_guard<std::mutex> pl(g_pool_mu);
    for (int p = 0; p < POOL; ++p) {
      if (g_pool[p]) D.StreamDestroy(g_pool[p]);
      if (g_join[p]) D.EventDestroy(g_join[p]);
      g_pool[p] = nullptr;
      g_join[p] = nullptr;
    }
    if (g_fork) D.EventDestroy(g_fork);
    g_fork = nullptr;
  }
  if (G.sum_buf) D.MemFree(G.sum_buf);
  G.sum_buf = 0;
  if (G.aot) D.ModuleUnload(G.aot);
  G.aot = nullptr;
  D.PrimaryCtxRelease(G.dev);
  G.ctx = nullptr;
  G.ordinal = -1;
  G.stream.store(nullptr);
  return JM_OK;
}

int jit_mat_run(int n, int dtype, int64_t batch, int64_t repeat, const void *in, void *out) {
  jm_run_desc d{n, dtype, JM_ADDEND_ONES, JM_KIND_SPECIALIZED, batch, repeat, in, out, nullptr, 0u};
  return run_impl(&d);
}

int jit_mat_run_ex(const jm_run_desc *d) { return run_impl(d); }

int jit_mat_run_many(const jm_run_desc *descs, int count, void *stream, unsigned flags) {
  return run_many_impl(descs, count, stream, flags);
}

int jit_mat_run_host(int n, int dtype, int64_t batch, int64_t repeat, const void *in, void *out) {
  jm_run_desc d{n, dtype, JM_ADDEND_ONES, JM_KIND_SPECIALIZED, batch, repeat, in, out, nullptr,
                JM_FLAG_HOST_BUFFERS};
  return run_impl(&d);
}

// Blob "JMC3": magic, the build digest of the library that compiled it (64
// hex chars: kernel source + planner + build defines, _build.py), key {n,
// dtype, addend}, entry count, then per compiled variant of the key (0
// resident, 1 streaming): variant, name expression, lowered symbol, cubin.
// Import accepts a blob only from the same build and only if each entry's
// name expression is the one this build would compile for the key, so the
// cubin always matches the plan it is launched with.
constexpr size_t DIGEST_LEN = 64;

int jit_mat_cache_export(int n, int dtype, int addend, void *buf, size_t cap, size_t *len) {
  int rc = check_key(n, dtype, addend, JM_KIND_SPECIALIZED);
  if (rc != JM_OK) return rc;
  if (!len) return fail(JM_E_INVALID, "NULL len");
  Slot *vs[2] = {&g_slots[JM_KIND_SPECIALIZED][addend][dtype][n], &g_stream_slots[addend][dtype][n]};
  std::unique_lock<std::mutex> l0(vs[0]->mu), l1(vs[1]->mu);
  bool have[2];
  std::string expr[2];
  size_t total = 4 + DIGEST_LEN + 3 * 4 + 4;
  int count = 0;
  for (int v = 0; v < 2; ++v) {
    have[v] = vs[v]->state.load(std::memory_order_acquire) == S_READY && !vs[v]->cubin.empty();
    if (!have[v]) continue;
    ++count;
    expr[v] = name_expression(n, dtype, addend, v == 1);
    total += 4 + 4 + expr[v].size() + 4 + vs[v]->lowered.size() + 8 + vs[v]->cubin.size();
  }
  if (!count)
    return fail(JM_E_INVALID, "key n=%d dtype=%d addend=%d is not compiled in this process", n, dtype, addend);
  *len = total;
  if (!buf) return JM_OK;
  if (cap < total) return fail(JM_E_INVALID, "buffer too small (%zu < %zu)", cap, total);
  char *p = (char *)buf;
  const int32_t key[3] = {n, dtype, addend};
  const int32_t cnt = count;
  memcpy(p, "JMC3", 4); p += 4;
  memcpy(p, jm_build_digest, DIGEST_LEN); p += DIGEST_LEN;
  memcpy(p, key, sizeof key); p += sizeof key;
  memcpy(p, &cnt, 4); p += 4;
  for (int v = 0; v < 2; ++v) {
    if (!have[v]) continue;
    const int32_t var = v;
    const uint32_t el = (uint32_t)expr[v].size();
    const uint32_t nl = (uint32_t)vs[v]->lowered.size();
    const uint64_t cl = (uint64_t)vs[v]->cubin.size();
    memcpy(p, &var, 4); p += 4;
    memcpy(p, &el, 4); p += 4;
    memcpy(p, expr[v].data(), el); p += el;
    memcpy(p, &nl, 4); p += 4;
    memcpy(p, vs[v]->lowered.data(), nl); p += nl;
    memcpy(p, &cl, 8); p += 8;
    memcpy(p, vs[v]->cubin.data(), cl); p += cl;
  }
  return JM_OK;
}

int jit_mat_cache_import(const void *blob, size_t len) {
  if (!blob || len < 4 + DIGEST_LEN + 12 + 4) return fail(JM_E_INVALID, "blob too short");
  if (!G.inited.load(std::memory_order_acquire)) return fail(JM_E_NOT_INITIALIZED, "jit_mat_init has not been called");
  const char *p = (const char *)blob, *end = p + len;
  if (memcmp(p, "JMC3", 4) != 0) return fail(JM_E_INVALID, "not a jitmat cubin blob");
  p += 4;
  if (memcmp(p, jm_build_digest, DIGEST_LEN) != 0)
    return fail(JM_E_INVALID, "blob from another library build (digest %.12s..., this build %.12s...)", p,
                (const char *)jm_build_digest);
  p += DIGEST_LEN;
  int32_t key[3], cnt;
  memcpy(key, p, sizeof key); p += sizeof key;
  memcpy(&cnt, p, 4); p += 4;
  int rc = check_key(key[0], key[1], key[2], JM_KIND_SPECIALIZED);
  if (rc != JM_OK) return rc;
  if (cnt < 1 || cnt > 2) return fail(JM_E_INVALID, "corrupt blob (entry count %d)", cnt);
  // parse and check every entry before installing any
  struct Entry { int32_t v; std::string sym; const char *cubin; uint64_t cl; };
  std::vector<Entry> es;
  auto str = [&](std::string &out) -> bool {
    uint32_t l;
    if ((size_t)(end - p) < 4) return false;
    memcpy(&l, p, 4); p += 4;
    if ((size_t)(end - p) < l) return false;
    out.assign(p, l); p += l;
    return true;
  };
  for (int i = 0; i < cnt; ++i) {
    Entry e{};
    std::string expr;
    if ((size_t)(end - p) < 4) return fail(JM_E_INVALID, "truncated blob");
    memcpy(&e.v, p, 4); p += 4;
    if (e.v < 0 || e.v > 1) return fail(JM_E_INVALID, "corrupt blob (variant %d)", e.v);
    if (!str(expr) || !str(e.sym) || (size_t)(end - p) < 8) return fail(JM_E_INVALID, "truncated blob");
    memcpy(&e.cl, p, 8); p += 8;
    if ((uint64_t)(end - p) < e.cl || e.cl == 0) return fail(JM_E_INVALID, "truncated blob");
    e.cubin = p; p += e.cl;
    const std::string want = name_expression(key[0], key[1], key[2], e.v == 1);
    if (expr != want)
      return fail(JM_E_INVALID, "blob entry %s does not match the key's kernel %s", expr.c_str(), want.c_str());
    es.push_back(std::move(e));
  }
  if (p != end) return fail(JM_E_INVALID, "trailing bytes in blob");
  for (const Entry &e : es) {
    Slot &s = e.v ? g_stream_slots[key[2]][key[1]][key[0]] : g_slots[JM_KIND_SPECIALIZED][key[2]][key[1]][key[0]];
    std::lock_guard<std::mutex> lk(s.mu);
    if (s.state.load(std::memory_order_acquire) == S_READY) continue;
    std::vector<char> cubin(e.cubin, e.cubin + e.cl);
    if ((rc = install_cubin(s, e.v ? OP_UPDATE_STREAM : OP_UPDATE, key[0], key[1], key[2], std::move(cubin), e.sym)) != JM_OK)
      return rc;
    s.compile_ms = 0.0;
    c_imports++;
    s.state.store(S_READY, std::memory_order_release);
  }
  return JM_OK;
}

int jit_mat_set_stream(void *cuda_stream) {
  G.stream.store(cuda_stream, std::memory_order_relaxed);
  return JM_OK;
}

int jit_mat_prepare(int n, int dtype, int addend, int kind) {
  Slot *s = nullptr;
  return lookup(n, dtype, addend, kind, &s);
}

int jit_mat_prepare_for(int n, int dtype, int addend, int kind, int64_t repeat, unsigned flags, int *variant) {
  int rc = check_key(n, dtype, addend, kind);
  if (rc != JM_OK) return rc;
  if (repeat < 0 || repeat > JM_REPEAT_MAX) return fail(JM_E_INVALID, "repeat must be in [0, 2^31)");
  // (the latency variant depends on the batch: prepared only when forced by JM_FLAG_LATENCY)
  jm_run_desc d{n, dtype, addend, kind, (int64_t)1 << 40, repeat, nullptr, nullptr, nullptr, flags};
  Slot *s = nullptr;
  if ((rc = lookup_run(d, &s)) != JM_OK) return rc;
  if (variant) *variant = variant_of(d);
  return JM_OK;
}

int jit_mat_dtype_from_name(const char *name) {
  if (!name) return fail(JM_E_INVALID, "NULL type name");
  if (strcmp(name, "float") == 0) return JM_F32;
  if (strcmp(name, "double") == 0) return JM_F64;
  return fail(JM_E_UNSUPPORTED, "%s not supported on the GPU path (float, double)", name);
}

const char *jit_mat_last_error(void) { return t_err.c_str(); }

int jit_mat_stats(jm_stats *out) {
  if (!out) return fail(JM_E_INVALID, "NULL stats");
  out->compilations = c_compilations.load();
  out->hits = c_hits.load();
  out->misses = c_misses.load();
  out->launches = c_launches.load();
  out->imports = c_imports.load();
  out->programs = c_programs.load();
  out->compile_ms_total = c_compile_us.load() / 1000.0;
  int ready = 0, failed = 0;
  for (int a = 0; a < NADD; ++a)
    for (int t = 0; t < NDT; ++t)
      for (int n = 1; n <= NMAX; ++n) {
        for (const Slot *sl : {&g_slots[JM_KIND_SPECIALIZED][a][t][n], &g_stream_slots[a][t][n]}) {
          const int st = sl->state.load();
          ready += st == S_READY;
          failed += st == S_FAILED;
        }
        if (n <= NLAT) {   // the latency variant's keys (tiny batches)
          const int st = g_lat_slots[a][t][n].state.load();
          ready += st == S_READY;
          failed += st == S_FAILED;
        }
      }
  out->keys_ready = ready;
  out->keys_failed = failed;
  return JM_OK;
}

}  // extern "C"
namespace {
// the JM_TILE_* code of a slot's plan (resident and streaming slots alike)
int tile_code(const jm::Plan &p) {
  return p.tile == (int)jm::Tile::TPM    ? JM_TILE_TPM
         : p.tile == (int)jm::Tile::Tpm2 ? JM_TILE_TPM2
         : p.tile == (int)jm::Tile::Tpms ? JM_TILE_TPMS
         : p.tile == (int)jm::Tile::Rows ? JM_TILE_ROWS
         : p.tile == (int)jm::Tile::F32Rows ? JM_TILE_F32_ROWS
         : p.tile == (int)jm::Tile::Reg ? JM_TILE_F64_REG
         : p.tile == (int)jm::Tile::F32Tc ? JM_TILE_F32_TC
         : p.tile == (int)jm::Tile::Dmma ? (p.w > 1 ? JM_TILE_CTA_DMMA : JM_TILE_WARP_DMMA)
                                         : (p.w > 1 ? JM_TILE_CTA_F32 : JM_TILE_WARP_F32);
}
}  // namespace
extern "C" {

int jit_mat_key_info(jm_key_info *keys, int cap) {
  int cnt = 0;
  for (int k = 0; k < NKIND; ++k)
    for (int a = 0; a < NADD; ++a)
      for (int t = 0; t < NDT; ++t)
        for (int n = 1; n <= NMAX; ++n) {
          Slot &s = g_slots[k][a][t][n];
          const int st = s.state.load(std::memory_order_acquire);
          if (st == S_EMPTY) continue;
          if (keys && cnt < cap) {
            jm_key_info &o = keys[cnt];
            o.n = n; o.dtype = t; o.addend = a; o.kind = k; o.state = st;
            o.regs = s.regs; o.local_bytes = s.local_bytes; o.smem_bytes = s.plan.smem;
            o.threads = s.plan.threads;
            o.tile = k == JM_KIND_GENERIC ? JM_TILE_GENERIC : tile_code(s.plan);
            o.cubin_bytes = s.cubin_bytes;
            o.compile_ms = s.compile_ms;
            o.op = 0;
            o.variant = 0;
          }
          ++cnt;
        }
  for (int a = 0; a < NADD; ++a)
    for (int t = 0; t < NDT; ++t)
      for (int n = 1; n <= NMAX; ++n) {
        Slot &s = g_stream_slots[a][t][n];
        const int st = s.state.load(std::memory_order_acquire);
        if (st == S_EMPTY) continue;
        if (keys && cnt < cap) {
          jm_key_info &o = keys[cnt];
          o.n = n; o.dtype = t; o.addend = a; o.kind = JM_KIND_SPECIALIZED; o.state = st;
          o.regs = s.regs; o.local_bytes = s.local_bytes; o.smem_bytes = s.plan.smem;
          o.threads = s.plan.threads;
          o.tile = tile_code(s.plan);
          o.cubin_bytes = s.cubin_bytes;
          o.compile_ms = s.compile_ms;
          o.op = 0;
          o.variant = 1;
        }
        ++cnt;
      }
  for (int a = 0; a < NADD; ++a)
    for (int t = 0; t < NDT; ++t)
      for (int n = 1; n <= NLAT; ++n) {
        Slot &s = g_lat_slots[a][t][n];
        const int st = s.state.load(std::memory_order_acquire);
        if (st == S_EMPTY) continue;
        if (keys && cnt < cap) {
          jm_key_info &o = keys[cnt];
          o.n = n; o.dtype = t; o.addend = a; o.kind = JM_KIND_SPECIALIZED; o.state = st;
          o.regs = s.regs; o.local_bytes = s.local_bytes; o.smem_bytes = s.plan.smem;
          o.threads = s.plan.threads;
          o.tile = JM_TILE_LAT;
          o.cubin_bytes = s.cubin_bytes;
          o.compile_ms = s.compile_ms;
          o.op = 0;
          o.variant = 2;
        }
        ++cnt;
      }
  for (int k = 0; k < 2; ++k)
    for (int t = 0; t < NDT; ++t)
      for (int n = 1; n <= NMAX; ++n) {
        Slot &s = g_mm_slots[k][t][n];
        const int st = s.state.load(std::memory_order_acquire);
        if (st == S_EMPTY || (k == JM_KIND_GENERIC)) continue;   // generic mm slots: always seeded
        if (keys && cnt < cap) {
          jm_key_info &o = keys[cnt];
          o.n = n; o.dtype = t; o.addend = 0; o.kind = k; o.state = st;
          o.regs = s.regs; o.local_bytes = s.local_bytes; o.smem_bytes = s.plan.smem;
          o.threads = s.plan.threads;
          o.tile = JM_TILE_MATMUL;
          o.cubin_bytes = s.cubin_bytes;
          o.compile_ms = s.compile_ms;
          o.op = 1;
          o.variant = 0;
        }
        ++cnt;
      }
  return cnt;
}

int jit_mat_reset_stats(void) {
  c_compilations = 0; c_hits = 0; c_misses = 0; c_launches = 0; c_compile_us = 0; c_imports = 0; c_programs = 0;
  return JM_OK;
}

int jit_mat_fill(int n, int dtype, int dist, uint64_t seed, int64_t global_first, int64_t batch, void *out) {
  int rc = check_key(n, dtype, JM_ADDEND_ONES, JM_KIND_SPECIALIZED);
  if (rc != JM_OK) return rc;
  if (dist < 0 || dist > 3) return fail(JM_E_INVALID, "dist %d invalid", dist);
  if (batch < 0 || global_first < 0) return fail(JM_E_INVALID, "negative batch/global_first");
  if (!G.inited.load()) return fail(JM_E_NOT_INITIALIZED, "jit_mat_init has not been called");
  if (batch == 0) return JM_OK;
  if (!out) return fail(JM_E_INVALID, "NULL buffer");
  if ((rc = ensure_ctx()) != JM_OK) return rc;
  long long total = (long long)batch * n * n, gf = global_first;
  unsigned long long sd = seed;
  int nn = n, ds = dist;
  CUdeviceptr p = (CUdeviceptr)out;
  void *args[] = {&p, &nn, &ds, &sd, &gf, &total};
  long long blocks = (total + 255) / 256;
  if (blocks > (long long)G.sms * 16) blocks = (long long)G.sms * 16;
  CUstream st = (CUstream)G.stream.load();
  CU_TRY(D.LaunchKernel(G.fill[dtype], (unsigned)blocks, 1, 1, 256, 1, 1, 0, st, args, nullptr), "cuLaunchKernel(fill)");
  c_launches++;
  return sync_if(0, st);
}

int jit_mat_checksum(int n, int dtype, int64_t global_first, int64_t batch, const void *x,
                     uint64_t *host_u64, double *host_f64) {
  int rc = check_key(n, dtype, JM_ADDEND_ONES, JM_KIND_SPECIALIZED);
  if (rc != JM_OK) return rc;
  if (batch < 0 || global_first < 0) return fail(JM_E_INVALID, "negative batch/global_first");
  if (!G.inited.load()) return fail(JM_E_NOT_INITIALIZED, "jit_mat_init has not been called");
  if (!host_u64 || !host_f64 || (batch > 0 && !x)) return fail(JM_E_INVALID, "NULL pointer");
  if ((rc = ensure_ctx()) != JM_OK) return rc;
  CUstream st = (CUstream)G.stream.load();
  CU_TRY(D.MemsetD8Async(G.sum_buf, 0, 16, st), "cuMemsetD8Async");
  long long total = (long long)batch * n * n, gf = global_first;
  if (total > 0) {
    int nn = n;
    CUdeviceptr px = (CUdeviceptr)x, pu = G.sum_buf, pf = G.sum_buf + 8;
    void *args[] = {&px, &nn, &gf, &total, &pu, &pf};
    long long blocks = (total + 255) / 256;
    if (blocks > (long long)G.sms * 8) blocks = (long long)G.sms * 8;
    CU_TRY(D.LaunchKernel(G.checksum[dtype], (unsigned)blocks, 1, 1, 256, 1, 1, 0, st, args, nullptr),
           "cuLaunchKernel(checksum)");
    c_launches++;
  }
  unsigned long long hv[2] = {0, 0};
  CU_TRY(D.MemcpyDtoHAsync(hv, G.sum_buf, 16, st), "cuMemcpyDtoHAsync(checksum)");
  CU_TRY(D.StreamSynchronize(st), "checksum");
  *host_u64 = hv[0];
  memcpy(host_f64, &hv[1], 8);
  return JM_OK;
}

int jit_mat_device_info(int *sm_count, int *cc_major, int *cc_minor) {
  if (!G.inited.load()) return fail(JM_E_NOT_INITIALIZED, "jit_mat_init has not been called");
  if (sm_count) *sm_count = G.sms;
  if (cc_major) *cc_major = G.cc_major;
  if (cc_minor) *cc_minor = G.cc_minor;
  return JM_OK;
}

const char *jit_mat_version(void) {
  static char buf[96];
  int maj = 0, min = 0;
  nvrtcVersion(&maj, &min);
  snprintf(buf, sizeof buf, "jitmat 0.1 (sm_100a; NVRTC %d.%d static)", maj, min);
  return buf;
}

// Test hook: NVRTC-compile a key without a device (no module load).  Lets the
// CPU-only test tier prove every specialization compiles for sm_100a.
int jit_mat_compile_check(int n, int dtype, int addend, long long *cubin_bytes) {
  int rc = JM_OK;
  std::string expr;
  if (addend == JM_OP_MASS) {   // n = dofs, dtype = quads
    if (n < 1 || dtype < 1 || n > jm::MASS_MAX || dtype > jm::MASS_MAX)
      return fail(JM_E_UNSUPPORTED, "dofs/quads must be in [1, %d]", jm::MASS_MAX);
    expr = mass_name_expression(n, dtype);
  } else {
    const bool op = addend == JM_OP_MATMUL || addend == JM_OP_STREAM || addend == JM_OP_LAT;
    rc = check_key(n, dtype, op ? JM_ADDEND_ONES : addend, JM_KIND_SPECIALIZED);
    if (rc != JM_OK) return rc;
    if (addend == JM_OP_STREAM && !jm::stream_ok(n, dtype))
      return fail(JM_E_UNSUPPORTED, "n=%d %s has no streaming variant", n, dtype == JM_F64 ? "double" : "float");
    if (addend == JM_OP_LAT && !jm::lat_ok(n))
      return fail(JM_E_UNSUPPORTED, "n=%d has no latency variant (n*n <= 32)", n);
    expr = addend == JM_OP_MATMUL   ? mm_name_expression(n, dtype)
           : addend == JM_OP_STREAM ? name_expression(n, dtype, JM_ADDEND_ONES, true)
           : addend == JM_OP_LAT    ? lat_name_expression(n, dtype, JM_ADDEND_ONES)
                                    : name_expression(n, dtype, addend);
  }
  std::vector<char> cubin;
  std::string lowered, log;
  rc = nvrtc_compile_expr(expr, cubin, lowered, log);
  if (rc != JM_OK) return fail(rc, "%s", log.c_str());
  if (cubin_bytes) *cubin_bytes = (long long)cubin.size();
  return JM_OK;
}

int jit_mat_matmul(int n, int dtype, int kind, int64_t batch, const void *a, const void *b, void *c,
                   void *stream) {
  int rc = check_key(n, dtype, JM_ADDEND_ONES, kind);
  if (rc != JM_OK) return rc;
  if (batch < 0) return fail(JM_E_INVALID, "batch must be >= 0 (got %lld)", (long long)batch);
  if (!G.inited.load(std::memory_order_acquire)) return fail(JM_E_NOT_INITIALIZED, "jit_mat_init has not been called");
  if (batch == 0) return JM_OK;
  if (!a || !b || !c) return fail(JM_E_INVALID, "NULL buffer");
  if (((unsigned long long)a | (unsigned long long)b | (unsigned long long)c) & 15)
    return fail(JM_E_ALIGN, "a/b/c must be 16-byte aligned");
  const unsigned long long bytes = (unsigned long long)batch * n * n * (dtype == JM_F64 ? 8 : 4);
  const unsigned long long pc = (unsigned long long)c;
  for (const void *p : {a, b}) {
    const unsigned long long q = (unsigned long long)p;
    if (q < pc + bytes && pc < q + bytes) return fail(JM_E_INVALID, "c must not overlap a or b");
  }
  Slot *s = nullptr;
  if ((rc = lookup_op(OP_MATMUL, n, dtype, JM_ADDEND_ONES, kind, &s)) != JM_OK) return rc;
  if ((rc = ensure_ctx()) != JM_OK) return rc;
  CUstream st = (CUstream)(stream ? stream : G.stream.load(std::memory_order_relaxed));
  const long long mpc = s->plan.mpc;
  const long long nchunks = (batch + mpc - 1) / mpc;
  unsigned grid = (unsigned)(nchunks < s->grid_cap ? nchunks : s->grid_cap);
  unsigned smem = (unsigned)s->plan.smem;
  const int es = dtype == JM_F64 ? 8 : 4;
  if (kind != JM_KIND_GENERIC && jm::mm_direct(batch, n, es)) {
    // small batch: the kernel's grid-wide direct path, no bulk-copy ring
    const long long blocks = (batch * n * n + jm::MM_THREADS - 1) / jm::MM_THREADS;
    grid = (unsigned)(blocks < jm::MM_DIRECT_GRID ? blocks : jm::MM_DIRECT_GRID);
    smem = 0;
  }
  CUdeviceptr pa = (CUdeviceptr)a, pb = (CUdeviceptr)b, pcc = (CUdeviceptr)c;
  long long bt = batch;
  int nn = n;
  void *args_spec[] = {&pa, &pb, &pcc, &bt};
  void *args_gen[] = {&pa, &pb, &pcc, &bt, &nn};
  CU_TRY(D.LaunchKernel(s->fn, grid, 1, 1, (unsigned)s->plan.threads, 1, 1, smem, st,
                        kind == JM_KIND_GENERIC ? args_gen : args_spec, nullptr),
         "cuLaunchKernel(matmul)");
  c_launches++;
  return sync_if(0, st);
}

int jit_mat_mass(int dofs, int quads, int kind, int64_t elements, const double *B, const double *op,
                 const double *x, double *y, void *stream) {
  if (dofs < 1 || quads < 1) return fail(JM_E_INVALID, "dofs and quads must be >= 1");
  if (dofs > jm::MASS_MAX || quads > jm::MASS_MAX)
    return fail(JM_E_UNSUPPORTED, "dofs/quads up to %d supported (got %d, %d)", jm::MASS_MAX, dofs, quads);
  if (kind != JM_KIND_SPECIALIZED && kind != JM_KIND_GENERIC)
    return fail(kind == JM_KIND_AOT_SPECIALIZED ? JM_E_UNSUPPORTED : JM_E_INVALID, "kind %d not available", kind);
  if (elements < 0) return fail(JM_E_INVALID, "elements must be >= 0");
  if (!G.inited.load(std::memory_order_acquire)) return fail(JM_E_NOT_INITIALIZED, "jit_mat_init has not been called");
  if (elements == 0) return JM_OK;
  if (!B || !op || !x || !y) return fail(JM_E_INVALID, "NULL buffer");
  if (((unsigned long long)op | (unsigned long long)x | (unsigned long long)y) & 15)
    return fail(JM_E_ALIGN, "op/x/y must be 16-byte aligned");
  const unsigned long long yb = (unsigned long long)elements * dofs * dofs * 8, py = (unsigned long long)y;
  const unsigned long long spans[3][2] = {{(unsigned long long)x, yb},
                                          {(unsigned long long)op, (unsigned long long)elements * quads * quads * 8},
                                          {(unsigned long long)B, (unsigned long long)dofs * quads * 8}};
  for (auto &sp : spans)
    if (sp[0] < py + yb && py < sp[0] + sp[1]) return fail(JM_E_INVALID, "y must not overlap B, op or x");
  Slot *s = nullptr;
  int rc = acquire_slot(g_mass_slots[kind][dofs][quads], OP_MASS, dofs, JM_F64, quads, kind, &s);
  if (rc != JM_OK) return rc;
  if ((rc = ensure_ctx()) != JM_OK) return rc;
  CUstream st = (CUstream)(stream ? stream : G.stream.load(std::memory_order_relaxed));
  const long long mpc = s->plan.mpc;
  const long long nchunks = (elements + mpc - 1) / mpc;
  const unsigned grid = (unsigned)(nchunks < s->grid_cap ? nchunks : s->grid_cap);
  CUdeviceptr pb = (CUdeviceptr)B, po = (CUdeviceptr)op, px = (CUdeviceptr)x, pyy = (CUdeviceptr)y;
  long long ne = elements;
  int dd = dofs, qq = quads;
  void *args_spec[] = {&pb, &po, &px, &pyy, &ne};
  void *args_gen[] = {&pb, &po, &px, &pyy, &ne, &dd, &qq};
  CU_TRY(D.LaunchKernel(s->fn, grid, 1, 1, (unsigned)s->plan.threads, 1, 1, (unsigned)s->plan.smem, st,
                        kind == JM_KIND_GENERIC ? args_gen : args_spec, nullptr),
         "cuLaunchKernel(mass)");
  c_launches++;
  return sync_if(0, st);
}

// Cache-hit cost of the key lookup (row a1), measured in C: `iters` lookups of
// an already-READY key, average nanoseconds per lookup into *ns.
int jit_mat_time_lookup(int n, int dtype, int addend, int kind, int64_t iters, double *ns) {
  if (!ns || iters <= 0) return fail(JM_E_INVALID, "bad arguments");
  Slot *s = nullptr;
  int rc = lookup(n, dtype, addend, kind, &s);   // make sure it is READY
  if (rc != JM_OK) return rc;
  const auto t0 = std::chrono::steady_clock::now();
  uintptr_t sink = 0;
  for (int64_t i = 0; i < iters; ++i) {
    rc = lookup(n, dtype, addend, kind, &s);
    sink += (uintptr_t)s + (uintptr_t)rc;
  }
  const double el = std::chrono::duration<double, std::nano>(std::chrono::steady_clock::now() - t0).count();
  *ns = el / (double)iters + (sink == 1 ? 1e-300 : 0.0);
  return JM_OK;
}

}  // extern "C"
