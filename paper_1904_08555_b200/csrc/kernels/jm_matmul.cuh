// jm_matmul.cuh — batched small matrix multiply-accumulate, the RAJA
// benchmark of PAPER.md §5.1 (Listing 8):
//
//     out[b](i,j) += in1[b](i,k) * in2[b](k,j)      (reading R16: per batch entry)
//
// specialized per (N, T) through NVRTC exactly like k_update (the paper wraps
// the loop nest in affine_jit_kernel_* so the RAJA range bounds become
// template arguments, Listing 9).  The work per matrix is 2N^3 flops against
// 4 N^2 elements of traffic (read A, B, C; write C), so at the paper's sizes
// (2x2, 8x8) it is HBM-bound: the kernel streams chunks of A and B through
// shared memory with 128-bit loads and gives every thread one output element,
// reading / writing C directly (coalesced: thread e owns element e).
// Appended to the NVRTC source after jm_update.cuh (no #include).
#ifndef JM_MATMUL_CUH
#define JM_MATMUL_CUH

namespace jm {

template <int N, class T>
__device__ __forceinline__ void matmul_body(const T *__restrict__ a, const T *__restrict__ b,
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

template <int N, class T>
__global__ void __launch_bounds__(MM_THREADS)
    k_matmul(const T *__restrict__ a, const T *__restrict__ b, T *__restrict__ c, long long batch) {
  matmul_body<N, T>(a, b, c, batch);
}

}  // namespace jm
#endif  // JM_MATMUL_CUH
