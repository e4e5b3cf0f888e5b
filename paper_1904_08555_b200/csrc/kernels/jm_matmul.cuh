// jm_matmul.cuh — batched small matrix multiply-accumulate, the RAJA
// benchmark of PAPER.md §5.1 (Listing 8):
//
//     out[b](i,j) += in1[b](i,k) * in2[b](k,j)      (reading R16: per batch entry)
//
// specialized per (N, T) through NVRTC exactly like k_update (the paper wraps
// the loop nest in affine_jit_kernel_* so the RAJA range bounds become
// template arguments, Listing 9).  The work per matrix is 2N^3 flops against
// 4 N^2 elements of traffic (read A, B, C; write C), so at the paper's sizes
// (2x2, 8x8) it is HBM-bound, and the kernel is a streaming pipeline:
//
//   * a persistent CTA owns every gridDim.x-th chunk of MPC matrices; a ring of
//     MM_STAGES shared-memory buffers holds the chunk's A, B and C, filled by
//     bulk copies (cp.async.bulk = the TMA engine, no tensor map needed for a
//     1-D copy) that signal an mbarrier with their byte count;
//   * one thread keeps the ring full; all threads wait on the stage's mbarrier,
//     compute C += A.B element-parallel out of shared memory (thread e owns
//     output element e of the chunk: conflict-free on B and C, broadcast on A),
//     and the updated C leaves through a bulk store, so loads, math and stores
//     of different chunks overlap with no register staging at all;
//   * the ragged tail (< MPC matrices, whose byte count need not be a multiple
//     of 16) is computed straight from global memory by one CTA.
//
// Batches with fewer full chunks than SMs take a direct grid-wide path
// (mm_direct, launched without the ring's shared memory).
// Sizes whose ring would not fit twice in shared memory (large odd N) keep the
// earlier staged loop (matmul_staged).  Appended to the NVRTC source after
// jm_update.cuh (no #include).
#ifndef JM_MATMUL_CUH
#define JM_MATMUL_CUH

namespace jm {

template <int N, class T>
__device__ __forceinline__ void matmul_staged(const T *__restrict__ a, const T *__restrict__ b,
                                            T *__restrict__ c, long long batch) {
  constexpr int NN = N * N, MPC = mm_mpc(N), NT = MM_THREADS, ES = sizeof(T);
  constexpr int MB = NN * ES;
  constexpr bool AL = ((MPC * MB) % 16) == 0;
  extern __shared__ __align__(16) char smem[];
  char *sa = smem;
  char *sb = smem + stage_bytes(MPC, N, ES);
  const int tid = threadIdx.x;
  const long long nchunks = (batch + MPC - 1) / MPC;
  for (long long ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
    const long long b0 = ch * MPC;
    const int cnt = (int)((batch - b0) < MPC ? (batch - b0) : MPC);
    // packed staging (stride MB), 128-bit when the chunk start is aligned
    stage_in<N, ES, MB, NT, AL>(reinterpret_cast<const char *>(a) + b0 * MB, sa, cnt, tid);
    stage_in<N, ES, MB, NT, AL>(reinterpret_cast<const char *>(b) + b0 * MB, sb, cnt, tid);
    __syncthreads();
    const T *A = reinterpret_cast<const T *>(sa);
    const T *B = reinterpret_cast<const T *>(sb);
    T *C = c + b0 * NN;
    const int total = cnt * NN;
    for (int e = tid; e < total; e += NT) {
      const int mi = e / NN, q = e - mi * NN, i = q / N, j = q - i * N;
      const T *Am = A + mi * NN + i * N;
      const T *Bm = B + mi * NN + j;
      T acc = C[e];
#pragma unroll
      for (int k = 0; k < N; ++k) acc = fmaT(Am[k], Bm[k * N], acc);
      C[e] = acc;
    }
    __syncthreads();
  }
}


// C[e] += (A.B)[e] for output element e of packed matrices
template <int N, class T, class PA, class PB, class PC>
__device__ __forceinline__ void mm_element(PA A, PB B, PC C, long long e) {
  constexpr int NN = N * N;
  const long long mi = e / NN;
  const int q = (int)(e - mi * NN), i = q / N, j = q - i * N;
  const T *Am = &A[mi * NN + i * N];
  const T *Bm = &B[mi * NN + j];
  T acc = C[e];
#pragma unroll
  for (int k = 0; k < N; ++k) acc = fmaT(Am[k], Bm[k * N], acc);
  C[e] = acc;
}
// ... for `total` elements, thread e owns element e
template <int N, class T, int NT, class PA, class PB, class PC>
__device__ __forceinline__ void mm_elements(PA A, PB B, PC C, int total, int tid) {
#pragma unroll 4
  for (int e = tid; e < total; e += NT) mm_element<N, T>(A, B, C, e);
}

template <int N, class T>
__device__ __forceinline__ void matmul_bulk(const T *__restrict__ a, const T *__restrict__ b, T *__restrict__ c,
                                            long long batch) {
  constexpr int ES = sizeof(T), NN = N * N, MB = NN * ES, NT = MM_THREADS;
  constexpr int MPC = mm_bulk_mpc(N, ES), ST = mm_bulk_stages(N, ES), CHB = MPC * MB;
  static_assert(CHB % 16 == 0, "bulk copies move multiples of 16 bytes");
  extern __shared__ __align__(128) char smem[];
  u64 *bar = reinterpret_cast<u64 *>(smem + ST * 3 * CHB);
  const int tid = threadIdx.x;
  const long long nfull = batch / MPC;
  const long long G = gridDim.x;
  const long long mine = nfull > blockIdx.x ? (nfull - 1 - blockIdx.x) / G + 1 : 0;
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < ST; ++s) mbar_init(bar + s, 1);
    fence_mbar_init();
  }
  __syncthreads();
  auto issue = [&](long long it, int s) {  // thread 0: chunk `it` of this CTA into stage s
    const size_t off = (size_t)(blockIdx.x + it * G) * CHB;
    char *st = smem + s * 3 * CHB;
    mbar_expect_tx(bar + s, 3 * CHB);
    bulk_g2s(st, reinterpret_cast<const char *>(a) + off, CHB, bar + s);
    bulk_g2s(st + CHB, reinterpret_cast<const char *>(b) + off, CHB, bar + s);
    bulk_g2s(st + 2 * CHB, reinterpret_cast<const char *>(c) + off, CHB, bar + s);
  };
  if (tid == 0)
    for (int s = 0; s < ST && s < mine; ++s) issue(s, s);
  int s = 0;
  unsigned phase = 0;
  for (long long it = 0; it < mine; ++it) {
    mbar_wait(bar + s, phase);
    char *st = smem + s * 3 * CHB;
    mm_elements<N, T, NT>(reinterpret_cast<const T *>(st), reinterpret_cast<const T *>(st + CHB),
                          reinterpret_cast<T *>(st + 2 * CHB), MPC * NN, tid);
    fence_proxy_async();
    __syncthreads();
    if (tid == 0) {
      bulk_s2g(reinterpret_cast<char *>(c) + (size_t)(blockIdx.x + it * G) * CHB, st + 2 * CHB, CHB);
      bulk_commit();
      if (it + ST < mine) {
        bulk_wait_read_all();  // the store has read stage s: refill it
        issue(it + ST, s);
      }
    }
    if (++s == ST) { s = 0; phase ^= 1u; }
  }
  // ragged tail: straight from global memory, by the CTA next in line
  const long long r0 = nfull * MPC;
  if (r0 < batch && blockIdx.x == (unsigned)(nfull % G))
    mm_elements<N, T, NT>(a + r0 * NN, b + r0 * NN, c + r0 * NN, (int)(batch - r0) * NN, tid);
  if (tid == 0) bulk_wait_all();
}

template <int N, class T>
__global__ void __launch_bounds__(MM_THREADS)
    k_matmul(const T *__restrict__ a, const T *__restrict__ b, T *__restrict__ c, long long batch) {
  if constexpr (mm_bulk(N, (int)sizeof(T))) {
    if (mm_direct(batch, N, (int)sizeof(T))) {  // small batch: whole grid, straight from global
      const long long total = batch * (N * N);
      for (long long e = (long long)blockIdx.x * MM_THREADS + threadIdx.x; e < total;
           e += (long long)gridDim.x * MM_THREADS)
        mm_element<N, T>(a, b, c, e);
    } else {
      matmul_bulk<N, T>(a, b, c, batch);
    }
  }
  else matmul_staged<N, T>(a, b, c, batch);
}

}  // namespace jm
#endif  // JM_MATMUL_CUH
