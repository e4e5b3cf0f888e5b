/*
 * jit_mat.h — C ABI of libjitmat: the batched, runtime-specialized Eigen
 * benchmark update of ClangJIT (Finkel, Poliakoff, Richards, arXiv 1904.08555)
 * on NVIDIA B200 (sm_100a).
 *
 * THE OPERATION (Listing 4, Listing 5 lines
 * 406-408):  for every matrix b in [0, batch)
 *
 *     M <- A + c * (M + M*M)      repeated `repeat` times,   c = T(0.00005)
 *
 * with A = Ones (the all-ones matrix the listings add; default) or, under the
 * prose reading of PAPER.md:362, A = I.  M*M is formed from the pre-update M
 * (Eigen evaluates products into a temporary).  There is no convergence early
 * exit.  T is float or double, chosen at run time by name like Listing 4's
 * test_aot(std::string &type, ...) and Listing 5's
 * test_jit.
 *
 * THE SPECIALIZATION (§2, §4 Algorithm 1 lines
 * 308-349, §4.1): the first call for a key {n, dtype, addend,
 * kind} instantiates the kernel template for that N and T through NVRTC —
 * from source embedded in the library, no file-system access (PAPER.md:83,
 * 351) — straight to an sm_100a cubin, loads it, and caches the function in a
 * process-global table (Algorithm 1 lines 319 and 347).  Later
 * calls with the same key hit the cache.  The GENERIC kind is a runtime-N
 * kernel compiled ahead of time (the analog of Listing 4's dynamic-size
 * path); it never compiles at run time.
 *
 * LAYOUT: `in` and `out` each hold `batch` matrices of n*n elements of type T,
 * contiguous, no padding between matrices (element (i,j) of matrix b at
 * b*n*n + i*n + j, or the column-major reading — both give the same buffer
 * result because f(M^T) = f(M)^T).
 *
 * OWNERSHIP: the library never allocates or frees caller memory and keeps no
 * reference to `in`/`out` after the work it enqueued completes.  `in == out`
 * (exact alias) is allowed; a partial overlap is JM_E_INVALID.
 *
 * ERRORS (an answer to PAPER.md:806, "no place to get out an error"): every
 * entry returns JM_OK (0) or a negative JM_E_* code; nothing aborts and no
 * exception crosses the ABI.  jit_mat_last_error() returns a thread-local
 * message (with the NVRTC log on JM_E_COMPILE).  Argument and compile errors
 * are detected before anything is enqueued.  Kernel faults are asynchronous
 * and surface at the caller's next synchronization, or at once with
 * JM_FLAG_SYNC / environment JIT_MAT_SYNC=1.  There is no CPU fallback: a
 * device that is not compute capability 10.x is JM_E_ARCH.
 *
 * THREADING: every function is thread-safe.  The first call for a key blocks
 * the calling host thread while it compiles (as __clang_jit does); concurrent
 * callers of the same key wait for that one compile; distinct keys compile in
 * parallel.  One process drives one device (jit_mat_init's).
 */
#ifndef JIT_MAT_H
#define JIT_MAT_H

#include <stddef.h>
#include <stdint.h>

#if defined(JM_BUILDING_LIB) && defined(__GNUC__)
#define JM_API __attribute__((visibility("default")))
#else
#define JM_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* element types: the names of Listing 4's type switch */
enum { JM_F32 = 0, JM_F64 = 1 };

/* addend A: the listings' Matrix::Ones (default) or the prose "I" */
enum { JM_ADDEND_ONES = 0, JM_ADDEND_IDENTITY = 1 };

/* kernel kind: the NVRTC-specialized template (Listing 5) or the AoT
 * runtime-N generic kernel (Listing 4) */
enum { JM_KIND_SPECIALIZED = 0, JM_KIND_GENERIC = 1,
       /* the same template compiled AHEAD of time by nvcc for Fig. 3's sizes
        * (n = 3, 7, 16, double): pre-seeded at init, never
        * compiled at run time; other keys -> JM_E_UNSUPPORTED */
       JM_KIND_AOT_SPECIALIZED = 2 };

/* status codes */
enum {
  JM_OK = 0,
  JM_E_INVALID = -1,          /* bad argument (n <= 0, batch < 0, repeat out of range, NULL, overlap) */
  JM_E_UNSUPPORTED = -2,      /* n > 64, dtype not f32/f64 ("long double"), unknown type name */
  JM_E_NOT_INITIALIZED = -3,  /* jit_mat_init not called, or after jit_mat_shutdown */
  JM_E_ARCH = -4,             /* device is not sm_100 (compute capability 10.x) */
  JM_E_COMPILE = -5,          /* NVRTC or module load failed, or the compiled kernel's plan cannot
                                  run on this device (shared memory, occupancy); log in
                                  jit_mat_last_error(); the key is then FAILED (not retried) */
  JM_E_CUDA = -6,             /* CUDA driver error (message in jit_mat_last_error()) */
  JM_E_ALIGN = -7             /* in/out not 16-byte aligned */
};

#define JM_N_MAX 64
#define JM_REPEAT_MAX 2147483647LL

/* run flags */
#define JM_FLAG_SYNC 1u          /* synchronize the stream before returning; report kernel faults */
#define JM_FLAG_HOST_BUFFERS 2u  /* in/out are HOST pointers: the library stages them through
                                    device buffers it owns, chunked and overlapped (see run_host) */
#define JM_FLAG_RESIDENT 4u      /* use the resident kernel whatever the repeat count (see VARIANT) */
#define JM_FLAG_STREAMING 8u     /* use the streaming kernel where the kind has one (see VARIANT) */
#define JM_FLAG_LATENCY 32u      /* use the latency kernel (a warp per matrix; n*n <= 32; see VARIANT) */
#define JM_FLAG_BATCH_COMPILE 16u /* jit_mat_run_many: compile the cold keys as a few NVRTC programs
                                    of several name expressions each (see jit_mat_run_many) */

/* Initialise for `device` (-1 = the calling thread's current CUDA device, else
 * device 0).  Loads the CUDA driver, retains the device's primary context (the
 * one PyTorch uses), checks compute capability 10.x (else JM_E_ARCH), loads the
 * ahead-of-time generic and auxiliary kernels and pre-seeds the generic cache
 * slots.  No NVRTC work.  Idempotent for the same device; a different device
 * while initialised is JM_E_INVALID. */
JM_API int jit_mat_init(int device);

/* out[b] = f^repeat(in[b]) for b in [0, batch): the specialized kernel for
 * (n, dtype), addend Ones, on the stream set by jit_mat_set_stream (default:
 * the legacy default stream).  `in`/`out` are device pointers (16-byte
 * aligned) on the initialised device.  n in [1, 64]; batch >= 0 (0: no-op);
 * repeat in [0, 2^31) (0: out is a bitwise copy of in).  Asynchronous.
 *
 * VARIANT (every specialized entry point): a call whose
 * repeat * (n + 1) is below the kind's measured switch point (jm_plan.h
 * stream_rn: 100..600 for f64 n >= 9 by tiling kind, 64 for f32 n = 9..16,
 * 140 for f32 n >= 17, for thread-per-matrix sizes (f64 n <= 7, f32 n <= 11)
 * only at f32 n = 3 with R >= 8 (their staged variant is selectable with
 * JM_FLAG_STREAMING), and not at f64 n = 16, R = 1; the HBM-bound side of the roofline and somewhat
 * beyond)
 * runs the STREAMING variant of the same specialization — the same tile code
 * behind a bulk-copy (TMA) ring, or for thread-per-matrix sizes behind a
 * double-buffered cp.async stage — which is
 * a second cache key, compiled on its first such call.  Results agree with the
 * resident kernel bit for bit (same arithmetic in the same order), except f64
 * n = 33, 34, where the resident kernel forms the thin border with DFMA, and
 * f64 n = 9, 10 and f32 n = 12..14, where the resident kernel is thread per
 * matrix with a staged product and the low-repeat one the DMMA / row-panel
 * ring (both within the parity bound).  Environment
 * JIT_MAT_STREAM=0/1 forces resident/streaming, JIT_MAT_STREAM_RN moves the
 * switch point (read once per process); per call, jm_run_desc.flags
 * JM_FLAG_RESIDENT / JM_FLAG_STREAMING force it.  A third, LATENCY variant
 * (a third cache key) serves tiny batches of n*n <= 32 matrices: when the batch
 * is at most 4 matrices per SM (or with JM_FLAG_LATENCY) each matrix gets a warp,
 * one element per lane, and the update's critical path is one n-long FMA chain
 * instead of a thread's n^2(n+1) FMAs (BASELINE.json configs[0], C1); it sums
 * in the thread-per-matrix kernel's order, so results agree bit for bit;
 * JIT_MAT_LATENCY=0 turns it off.  JIT_MAT_DUMP_CUBIN=<dir> (inspection only)
 * writes each NVRTC cubin to <dir>/<symbol>.cubin. */
JM_API int jit_mat_run(int n, int dtype, int64_t batch, int64_t repeat, const void *in, void *out);

/* Unload every module, drop the cache and release the primary context.  Later
 * calls return JM_E_NOT_INITIALIZED until jit_mat_init is called again. */
JM_API int jit_mat_shutdown(void);

/* ---- extensions ---------------------------------------------------------- */

typedef struct {
  int n, dtype, addend, kind;
  int64_t batch, repeat;
  const void *in;
  void *out;
  void *stream;      /* CUstream / cudaStream_t; NULL = the stream set by jit_mat_set_stream */
  unsigned flags;    /* JM_FLAG_* */
} jm_run_desc;

/* General entry: any addend / kind / stream / flags.  With JM_FLAG_HOST_BUFFERS
 * `in`/`out` are host pointers (pinned or pageable) and the call is
 * synchronous: the input streams host->device in chunks, each chunk is updated
 * on the device, and results stream back, with copies and compute overlapped on
 * library-owned streams and staging buffers. */
JM_API int jit_mat_run_ex(const jm_run_desc *d);

/* Convenience for the host-buffer path = run_ex(kind SPECIALIZED, addend Ones,
 * JM_FLAG_HOST_BUFFERS).  Synchronous. */
JM_API int jit_mat_run_host(int n, int dtype, int64_t batch, int64_t repeat, const void *in, void *out);

/* Mixed-N batch (BASELINE.json configs[3]): `count` independent groups, each a
 * device-buffer descriptor with its own n / dtype / addend / kind / batch /
 * repeat (the per-descriptor `stream` and JM_FLAG_HOST_BUFFERS are not allowed).
 * All cold keys are specialized first, concurrently on host threads (distinct
 * keys compile in parallel, "roughly additive" compile times
 * become overlapped); then the groups are launched concurrently on a pool of
 * library streams forked from and joined back into `stream` (NULL = the set
 * stream), so small groups fill the GPU together.  Asynchronous w.r.t. the
 * host unless `flags` has JM_FLAG_SYNC.  Every descriptor is validated before
 * anything is compiled or launched.  With JM_FLAG_BATCH_COMPILE the cold keys
 * are instead split into G groups (environment JIT_MAT_COMPILE_GROUPS, default
 * the host's hardware threads) and each group is ONE NVRTC program with a name
 * expression per key, so the embedded template source is parsed G times rather
 * than once per key. */
JM_API int jit_mat_run_many(const jm_run_desc *descs, int count, void *stream, unsigned flags);

/* Share specializations between processes (the paper's
 * compile-time concern).  jit_mat_cache_export writes a
 * self-describing blob ("JMC3": the library's build digest, the key, and per
 * compiled variant — resident and/or streaming — the name expression, kernel
 * symbol and sm_100a cubin) of a specialized key into
 * `buf` (`cap` bytes); `*len` receives the blob size (pass buf = NULL to
 * query).  JM_E_INVALID if neither variant of the key has been compiled.
 * jit_mat_cache_import installs such a blob (from the same library build) for
 * its key without running NVRTC: one rank compiles, broadcasts the blob, the
 * other ranks import it.  Importing into a READY slot is a no-op (JM_OK); a
 * blob from another build (digest mismatch), an entry whose name expression is
 * not the one this build compiles for the key, or a corrupt blob is
 * JM_E_INVALID. */
JM_API int jit_mat_cache_export(int n, int dtype, int addend, void *buf, size_t cap, size_t *len);
JM_API int jit_mat_cache_import(const void *blob, size_t len);

/* Batched small matrix multiply-accumulate, the RAJA benchmark of PAPER.md
 * §5.1 (Listing 8):
 *     c[b] += a[b] * b[b]        for b in [0, batch)
 * each a n x n row-major matrix of `dtype` (Listing 8's MAT2D(r,c,size) =
 * r*size + c), contiguous per batch.  kind JM_KIND_SPECIALIZED instantiates
 * jm::k_matmul<n, T> through NVRTC on first use (cached like jit_mat_run);
 * JM_KIND_GENERIC is the runtime-n kernel.  Device pointers, 16-byte aligned; c
 * must not overlap a or b (a and b may alias each other).  Asynchronous on
 * `stream` (NULL = the set stream).  As printed, Listing 8's lambda ignores the
 * batch index and accumulates every entry into one output; the batched form is
 * the evident intent (reading R16). */
JM_API int jit_mat_matmul(int n, int dtype, int kind, int64_t batch, const void *a, const void *b,
                          void *c, void *stream);

/* Laghos 2D mass-operator action rMassMultAdd2D<NUM_DOFS_1D, NUM_QUAD_1D>
 * (§5.3, Listing 12, Fig. 7; SURVEY.md §8(f) f4;
 * DESIGN.md reading R18), FP64, for each element e in [0, elements):
 *     S = (B X_e B^T) .* op_e ;   y_e += B^T S B
 * B: quads x dofs row-major (Laghos' dofToQuad; its transpose is quadToDof),
 * op: elements x quads x quads, x and y: elements x dofs x dofs, all row-major
 * doubles, device pointers (op/x/y 16-byte aligned; y must not overlap B, op
 * or x).  kind JM_KIND_SPECIALIZED instantiates jm::k_mass<dofs, quads>
 * through NVRTC (replacing Laghos' ~32-entry dispatch map of explicit
 * instantiations, Listing 12) — for the larger (dofs, quads) a warp per
 * element with the contractions on the FP64 tensor cores (DESIGN.md §10 f4);
 * the summation order differs from the CPU oracle's (parity is relative to the
 * contraction's magnitude scale).  JM_KIND_GENERIC is the runtime-(dofs, quads)
 * kernel.  1 <= dofs, quads <= 8 (Fig. 7's d, q in {2, 4, 8}); larger is
 * JM_E_UNSUPPORTED.  Asynchronous on `stream` (NULL = the set stream). */
JM_API int jit_mat_mass(int dofs, int quads, int kind, int64_t elements, const double *B,
                        const double *op, const double *x, double *y, void *stream);

/* Stream used by jit_mat_run (e.g. torch.cuda.current_stream().cuda_stream). */
JM_API int jit_mat_set_stream(void *cuda_stream);

/* Look up (and on a miss, compile and load) the kernel for a key without
 * launching.  The analog of forcing an instantiation ahead of use. */
JM_API int jit_mat_prepare(int n, int dtype, int addend, int kind);

/* As jit_mat_prepare, but for the kernel a run with this `repeat` and `flags`
 * (JM_FLAG_RESIDENT / JM_FLAG_STREAMING honoured) would launch — the resident
 * or the streaming variant, see jit_mat_run; `*variant` (may be NULL)
 * receives 0 (resident) or 1 (streaming). */
JM_API int jit_mat_prepare_for(int n, int dtype, int addend, int kind, int64_t repeat, unsigned flags,
                               int *variant);

/* "float" -> JM_F32, "double" -> JM_F64; "long double" and anything else ->
 * JM_E_UNSUPPORTED (the GPU path supports two of Listing 4's three types). */
JM_API int jit_mat_dtype_from_name(const char *name);

/* Thread-local description of the last error on this thread ("" if none). */
JM_API const char *jit_mat_last_error(void);

/* Cache statistics (SPEC.md:540-545 analog). */
typedef struct {
  int64_t compilations;      /* NVRTC compiles performed (successful or not) */
  int64_t hits;              /* lookups answered from the cache */
  int64_t misses;            /* lookups that had to compile (or wait for a compile) */
  int64_t launches;          /* kernels launched by this library */
  double compile_ms_total;   /* wall time inside NVRTC + module load */
  int32_t keys_ready;        /* specialized update cache slots (resident, streaming or latency variant) in READY state */
  int32_t keys_failed;       /* cache slots in FAILED state */
  int64_t imports;           /* keys installed by jit_mat_cache_import (no NVRTC) */
  int64_t programs;          /* NVRTC programs of batched compiles (JM_FLAG_BATCH_COMPILE) */
} jm_stats;

typedef struct {
  int32_t n, dtype, addend, kind;
  int32_t state;             /* 0 empty, 1 compiling, 2 ready, 3 failed */
  int32_t regs;              /* CU_FUNC_ATTRIBUTE_NUM_REGS (the Fig. 5 analog) */
  int32_t local_bytes;       /* CU_FUNC_ATTRIBUTE_LOCAL_SIZE_BYTES (spills) */
  int32_t smem_bytes;        /* dynamic shared memory per CTA of the launch plan */
  int32_t threads;           /* threads per CTA of the launch plan */
  int32_t tile;              /* tiling kind (JM_TILE_*) chosen by the planner */
  int64_t cubin_bytes;
  double compile_ms;
  int32_t op;                /* 0 = update (jit_mat_run), 1 = multiply-accumulate (jit_mat_matmul) */
  int32_t variant;           /* update: 0 resident kernel, 1 streaming (low-repeat) kernel */
} jm_key_info;

/* tiling kinds reported in jm_key_info.tile */
enum { JM_TILE_GENERIC = 0, JM_TILE_TPM = 1, JM_TILE_WARP_DMMA = 2, JM_TILE_CTA_DMMA = 3,
       JM_TILE_WARP_F32 = 4, JM_TILE_CTA_F32 = 5, JM_TILE_ROWS = 6, JM_TILE_MATMUL = 7,
       JM_TILE_TPM2 = 8 /* two threads per matrix (FP64 n = 8) */,
       JM_TILE_TPMS = 9 /* thread per matrix, product staged in shared memory (FP64 n = 9, 10, FP32 12..14) */,
       JM_TILE_F32_ROWS = 10 /* FP32 row panels: 4 threads per matrix own full rows (n = 15, 16) */,
       JM_TILE_F64_REG = 11 /* FP64 register tiles with DFMA (sizes DMMA pads badly) */,
       JM_TILE_LAT = 12 /* latency kernel: a warp per matrix, an element per lane (tiny batches) */,
       JM_TILE_F32_TC = 13 /* FP32 on the tensor cores: m16n8k8 TF32 mma, operands split hi + lo (3xTF32; n = 32 and 37..64, zero-padded to a multiple of 8) */ };

JM_API int jit_mat_stats(jm_stats *out);
/* Copy up to `cap` non-empty slots into `keys`; returns the number of
 * non-empty slots (may exceed cap). */
JM_API int jit_mat_key_info(jm_key_info *keys, int cap);
/* Reset counters (not the cache). */
JM_API int jit_mat_reset_stats(void);

/* ---- driver support (untimed plumbing) ----------- */

/* Fill out[0 .. batch*n*n) on the device with the counter-hash input generator
 * keyed by the GLOBAL matrix index (global_first + b), so a batch split across
 * ranks equals the unsplit batch.  dist: 0 paper (iota), 1 bench (U[-1,1)),
 * 2 hard (U[0,1) * 2*4000/n), 3 signed hard (U[-1,1) * 2*4000/n).  The definition is written out in
 * jm_synth/__init__.py (host side); this is an independent device
 * implementation of the same definition.  Asynchronous on the set stream. */
JM_API int jit_mat_fill(int n, int dtype, int dist, uint64_t seed, int64_t global_first,
                 int64_t batch, void *out);

/* Order-independent checksum of x[0 .. batch*n*n):
 *   S = sum_e splitmix64(bits(x_e) ^ PHI*(global_first*n*n + e)) mod 2^64,
 * plus the plain f64 sum.  Synchronous; results written to host pointers. */
JM_API int jit_mat_checksum(int n, int dtype, int64_t global_first, int64_t batch, const void *x,
                     uint64_t *host_u64, double *host_f64);

/* Device / library facts: SM count, CC major/minor, library version string. */
JM_API int jit_mat_device_info(int *sm_count, int *cc_major, int *cc_minor);
JM_API const char *jit_mat_version(void);

/* ---- test hook ------------------------------------------------------------ */

/* NVRTC-compile the specialized kernel for a key to an sm_100a cubin WITHOUT a
 * device or jit_mat_init (nothing is loaded or cached).  Lets a CPU-only test
 * tier prove that every specialization compiles.  addend = JM_OP_MATMUL selects
 * the multiply-accumulate template instead.  cubin_bytes may be NULL. */
#define JM_OP_MATMUL 2
#define JM_OP_MASS 3     /* compile_check(dofs, quads, JM_OP_MASS, ...): k_mass<dofs, quads> */
#define JM_OP_STREAM 4   /* the streaming (low-repeat) variant of the update (addend Ones) */
#define JM_OP_LAT 5      /* the latency variant of the update (addend Ones; n*n <= 32) */
JM_API int jit_mat_compile_check(int n, int dtype, int addend, long long *cubin_bytes);

/* Cache-hit cost of the key lookup (the paper calls the
 * lookup overhead "noticeable", and dominant for small work,
 * PAPER.md:560): `iters` lookups of a READY key (compiled first if needed),
 * average nanoseconds per lookup written to *ns. */
JM_API int jit_mat_time_lookup(int n, int dtype, int addend, int kind, int64_t iters, double *ns);

#ifdef __cplusplus
}
#endif
#endif /* JIT_MAT_H */
