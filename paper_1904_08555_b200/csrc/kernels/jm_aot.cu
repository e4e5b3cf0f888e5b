// jm_aot.cu — kernels compiled AHEAD OF TIME by nvcc into an sm_100a cubin
// that libjitmat embeds and loads at jit_mat_init:
//
//   * the GENERIC runtime-N update — the analog of Listing 4's
//     Matrix<T,Dynamic,Dynamic> path: the same recurrence,
//     but N is a kernel argument, so every loop bound is a runtime value and the
//     matrices live in shared memory (Eigen's dynamic matrices live on the
//     heap, PAPER.md:468 footnote).  This is the un-specialized comparison
//     (Figs. 3-4).  It is deliberately a fair kernel, not a
//     strawman: coalesced staging, several matrices per CTA for small N.
//   * fill / checksum — driver plumbing.
#include "jm_plan.h"
#include "jm_update.cuh"
#include "jm_matmul.cuh"
#include "jm_mass.cuh"

namespace jm {

template <class T, Addend A>
__device__ __forceinline__ void generic_update(const T *__restrict__ in, T *__restrict__ out,
                                               long long batch, int repeat, int n) {
  constexpr int NT = GENERIC_THREADS;
  const int nn = n * n;
  const int mpc = generic_mpc(n);
  extern __shared__ __align__(16) char smem[];
  T *M = reinterpret_cast<T *>(smem);
  T *P = M + mpc * nn;
  const T c = T(0.00005);
  const int tid = threadIdx.x;
  const long long nchunks = (batch + mpc - 1) / mpc;
  for (long long ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
    const long long b0 = ch * mpc;
    const int cnt = (int)((batch - b0) < mpc ? (batch - b0) : mpc);
    const int total = cnt * nn;
    for (int e = tid; e < total; e += NT) M[e] = in[b0 * nn + e];
    __syncthreads();
    for (int r = 0; r < repeat; ++r) {
      for (int e = tid; e < total; e += NT) {
        const int mi = e / nn, q = e - mi * nn, i = q / n, j = q - i * n;
        const T *Mm = M + mi * nn;
        T acc = Mm[q];
        for (int k = 0; k < n; ++k) acc = fmaT(Mm[i * n + k], Mm[k * n + j], acc);
        P[e] = acc;
      }
      __syncthreads();
      for (int e = tid; e < total; e += NT) {
        const int q = e % nn, i = q / n, j = q - i * n;
        M[e] = (A == Addend::Ones || i == j) ? fmaT(c, P[e], T(1)) : c * P[e];
      }
      __syncthreads();
    }
    for (int e = tid; e < total; e += NT) out[b0 * nn + e] = M[e];
    __syncthreads();
  }
}

// Generic (runtime-N) batched multiply-accumulate: the un-specialized
// comparison for matmul_body (same staging, runtime loop bounds).
template <class T>
__device__ __forceinline__ void matmul_generic(const T *__restrict__ a, const T *__restrict__ b,
                                               T *__restrict__ c, long long batch, int n) {
  constexpr int NT = MM_THREADS;
  const int nn = n * n, mpc = mm_mpc(n);
  extern __shared__ __align__(16) char smem[];
  T *A = reinterpret_cast<T *>(smem);
  T *B = reinterpret_cast<T *>(smem + stage_bytes(mpc, n, (int)sizeof(T)));
  const int tid = threadIdx.x;
  const long long nchunks = (batch + mpc - 1) / mpc;
  for (long long ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
    const long long b0 = ch * mpc;
    const int cnt = (int)((batch - b0) < mpc ? (batch - b0) : mpc);
    const int total = cnt * nn;
    for (int e = tid; e < total; e += NT) {
      A[e] = a[b0 * nn + e];
      B[e] = b[b0 * nn + e];
    }
    __syncthreads();
    T *C = c + b0 * nn;
    for (int e = tid; e < total; e += NT) {
      const int mi = e / nn, q = e - mi * nn, i = q / n, j = q - i * n;
      T acc = C[e];
      for (int k = 0; k < n; ++k) acc = fmaT(A[mi * nn + i * n + k], B[mi * nn + k * n + j], acc);
      C[e] = acc;
    }
    __syncthreads();
  }
}

// Generic (runtime D, Q) Laghos mass action: the non-specialized comparison of
// Fig. 7 — same algorithm as mass_body with runtime loop
// bounds, so the per-element quadrature array lives in local memory.
__device__ __forceinline__ void mass_generic(const double *__restrict__ B, const double *__restrict__ op,
                                             const double *__restrict__ x, double *__restrict__ y,
                                             long long elements, int D, int Q) {
  constexpr int NT = MASS_THREADS, MPC = MASS_THREADS;
  extern __shared__ __align__(16) char smem[];
  double *sx = reinterpret_cast<double *>(smem);
  double *sy = sx + MPC * D * D;
  double *so = sy + MPC * D * D;
  double *sB = so + MPC * Q * Q;
  const int tid = threadIdx.x;
  for (int i = tid; i < Q * D; i += NT) sB[i] = B[i];
  const long long nchunks = (elements + MPC - 1) / MPC;
  for (long long ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
    const long long e0 = ch * MPC;
    const int cnt = (int)((elements - e0) < MPC ? (elements - e0) : MPC);
    for (int i = tid; i < cnt * D * D; i += NT) {
      sx[i] = x[e0 * D * D + i];
      sy[i] = y[e0 * D * D + i];
    }
    for (int i = tid; i < cnt * Q * Q; i += NT) so[i] = op[e0 * Q * Q + i];
    __syncthreads();
    if (tid < cnt) {
      const double *X = sx + tid * D * D, *O = so + tid * Q * Q;
      double *Y = sy + tid * D * D;
      double S[MASS_MAX * MASS_MAX], sol[MASS_MAX];
      for (int i = 0; i < Q * Q; ++i) S[i] = 0.0;
      for (int dy = 0; dy < D; ++dy) {
        for (int qx = 0; qx < Q; ++qx) sol[qx] = 0.0;
        for (int dx = 0; dx < D; ++dx)
          for (int qx = 0; qx < Q; ++qx) sol[qx] = fmaT(sB[qx * D + dx], X[dy * D + dx], sol[qx]);
        for (int qy = 0; qy < Q; ++qy)
          for (int qx = 0; qx < Q; ++qx) S[qy * Q + qx] = fmaT(sB[qy * D + dy], sol[qx], S[qy * Q + qx]);
      }
      for (int i = 0; i < Q * Q; ++i) S[i] *= O[i];
      for (int qy = 0; qy < Q; ++qy) {
        for (int dx = 0; dx < D; ++dx) sol[dx] = 0.0;
        for (int qx = 0; qx < Q; ++qx)
          for (int dx = 0; dx < D; ++dx) sol[dx] = fmaT(sB[qx * D + dx], S[qy * Q + qx], sol[dx]);
        for (int dy = 0; dy < D; ++dy)
          for (int dx = 0; dx < D; ++dx) Y[dy * D + dx] = fmaT(sB[qy * D + dy], sol[dx], Y[dy * D + dx]);
      }
    }
    __syncthreads();
    for (int i = tid; i < cnt * D * D; i += NT) y[e0 * D * D + i] = sy[i];
    __syncthreads();
  }
}

__device__ __forceinline__ u64 splitmix64(u64 z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}

// Input generator (definition: jm_synth/__init__.py docstring).  Every
// floating-point step is an explicit round-to-nearest intrinsic so the device
// reproduces the host's numpy arithmetic bit for bit (no FMA contraction).
template <class T>
__device__ __forceinline__ void fill_impl(T *__restrict__ out, int n, int dist, u64 seed,
                                          long long gfirst, long long total) {
  const long long nn = (long long)n * n;
  const double scale = __ddiv_rn(8000.0, (double)n);
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    double x;
    if (dist == 0) {
      x = (double)(e % nn);
    } else {
      const u64 ge = (u64)(gfirst * nn + e);
      const u64 z = splitmix64(seed ^ (0x9E3779B97F4A7C15ull * (ge + 1ull)));
      const double u = __dmul_rn((double)(z >> 11), 1.1102230246251565e-16);  // 2^-53
      x = (dist == 1)   ? __dsub_rn(__dmul_rn(2.0, u), 1.0)
          : (dist == 2) ? __dmul_rn(u, scale)
                        : __dmul_rn(__dsub_rn(__dmul_rn(2.0, u), 1.0), scale);   // 3: signed hard
    }
    if constexpr (sizeof(T) == 8) out[e] = x;
    else out[e] = __double2float_rn(x);
  }
}

template <class T>
__device__ __forceinline__ void checksum_impl(const T *__restrict__ x, int n, long long gfirst,
                                              long long total, u64 *res_u64, double *res_f64) {
  const u64 base = (u64)(gfirst * (long long)n * n);
  u64 h = 0;
  double s = 0.0;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    u64 bits;
    if constexpr (sizeof(T) == 8) bits = (u64)__double_as_longlong(x[e]);
    else bits = (u64)__float_as_uint(x[e]);
    h += splitmix64(bits ^ (0x9E3779B97F4A7C15ull * (base + (u64)e)));
    s += (double)x[e];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    h += __shfl_xor_sync(0xffffffffu, h, o);
    s += __shfl_xor_sync(0xffffffffu, s, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(reinterpret_cast<unsigned long long *>(res_u64), (unsigned long long)h);
    atomicAdd(res_f64, s);
  }
}

}  // namespace jm

#define JM_GENERIC(NAME, T, ADD)                                                              \
  extern "C" __global__ void __launch_bounds__(jm::GENERIC_THREADS)                            \
      NAME(const T *__restrict__ in, T *__restrict__ out, long long batch, int repeat, int n) { \
    jm::generic_update<T, ADD>(in, out, batch, repeat, n);                                     \
  }
JM_GENERIC(jm_generic_f32_ones, float, jm::Addend::Ones)
JM_GENERIC(jm_generic_f32_identity, float, jm::Addend::Identity)
JM_GENERIC(jm_generic_f64_ones, double, jm::Addend::Ones)
JM_GENERIC(jm_generic_f64_identity, double, jm::Addend::Identity)

// AoT SPECIALIZATIONS ("explicit
// specializations ... are used instead", Fig. 3 "AoT specialization" bar,
// PAPER.md:440-466): the very same template body the NVRTC path instantiates,
// compiled here by nvcc for the sizes of Fig. 3 (3, 7, 16) in double, so the
// three-way comparison JIT / AoT-specialization / AoT-generic can be made.
#define JM_AOT_SPEC(N, T, TN, ADD, AN)                                                           \
  extern "C" __global__ void __launch_bounds__(jm::plan_specialized(N, TN).threads)              \
      jm_aotspec_##T##_n##N##_##AN(const T *__restrict__ in, T *__restrict__ out, long long batch, \
                                   int repeat) {                                                 \
    jm::update_body<N, T, ADD, jm::tile_for(N, TN)>(in, out, batch, repeat);                     \
  }
JM_AOT_SPEC(3, double, 1, jm::Addend::Ones, ones)
JM_AOT_SPEC(7, double, 1, jm::Addend::Ones, ones)
JM_AOT_SPEC(16, double, 1, jm::Addend::Ones, ones)
JM_AOT_SPEC(3, double, 1, jm::Addend::Identity, identity)
JM_AOT_SPEC(7, double, 1, jm::Addend::Identity, identity)
JM_AOT_SPEC(16, double, 1, jm::Addend::Identity, identity)

extern "C" __global__ void __launch_bounds__(jm::MM_THREADS)
    jm_mm_generic_f32(const float *__restrict__ a, const float *__restrict__ b, float *__restrict__ c,
                      long long batch, int n) {
  jm::matmul_generic<float>(a, b, c, batch, n);
}
extern "C" __global__ void __launch_bounds__(jm::MM_THREADS)
    jm_mm_generic_f64(const double *__restrict__ a, const double *__restrict__ b, double *__restrict__ c,
                      long long batch, int n) {
  jm::matmul_generic<double>(a, b, c, batch, n);
}

extern "C" __global__ void __launch_bounds__(jm::MASS_THREADS)
    jm_mass_generic(const double *__restrict__ B, const double *__restrict__ op, const double *__restrict__ x,
                    double *__restrict__ y, long long elements, int D, int Q) {
  jm::mass_generic(B, op, x, y, elements, D, Q);
}

extern "C" __global__ void jm_fill_f32(float *out, int n, int dist, unsigned long long seed,
                                       long long gfirst, long long total) {
  jm::fill_impl<float>(out, n, dist, seed, gfirst, total);
}
extern "C" __global__ void jm_fill_f64(double *out, int n, int dist, unsigned long long seed,
                                       long long gfirst, long long total) {
  jm::fill_impl<double>(out, n, dist, seed, gfirst, total);
}
extern "C" __global__ void jm_checksum_f32(const float *x, int n, long long gfirst, long long total,
                                           unsigned long long *ru, double *rf) {
  jm::checksum_impl<float>(x, n, gfirst, total, ru, rf);
}
extern "C" __global__ void jm_checksum_f64(const double *x, int n, long long gfirst, long long total,
                                           unsigned long long *ru, double *rf) {
  jm::checksum_impl<double>(x, n, gfirst, total, ru, rf);
}
