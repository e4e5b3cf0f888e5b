// lds_wavefronts.cu — cost of one LDS.128 / LDS.64 warp instruction on sm_100a
// under the broadcast patterns the FP32 tile kernels produce (r02 redesign).
// Unlike lds_patterns.cu (r01), whose loop issued ~9 ALU instructions per load
// and so measured the issue rate, the timed loop here is 16 independent
// loads per iteration from precomputed addresses plus one IADD each, so the
// LSU (not the issue slot) is the bottleneck.  Run plain for the rate and
// under ncu for wavefronts per instruction:
//   ncu --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,smsp__inst_executed_op_shared_ld.sum ./lds_wavefronts
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lds_wavefronts lds_wavefronts.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITER = 4096;

// byte offset (within a 16 KB window) that lane reads, per pattern
__device__ __forceinline__ unsigned pat_off(int pat, int lane, int bytes) {
  switch (pat) {
    case 0: return lane * bytes;                 // 32 distinct consecutive
    case 1: return 0;                            // broadcast
    case 2: return (lane % 8) * bytes;           // 8 distinct, each quarter reads all 8
    case 3: return (lane / 4) * bytes;           // 8 distinct, 4 consecutive lanes share
    case 4: return (lane / 8) * bytes;           // 4 distinct, one per quarter
    case 5: return (lane % 4) * bytes;           // 4 distinct, all in each quarter
    case 6: return (lane % 16) * bytes;          // 16 distinct consecutive
    case 7: return (lane / 2) * bytes;           // 16 distinct, pairs share
    case 8: return (lane / 4) * 144;             // 8 rows, odd-16B row stride 144 B (LDM/4 odd)
    case 9: return (lane % 4) * 144 + (lane / 16) * 4608;   // 4 rows x 2 matrices
    case 10: return (lane / 8) * 4608 + (lane % 8 / 4) * bytes;  // 4 matrices x 2 chunks
    default: return (lane % 8) * 2 * bytes;      // 8 distinct at 2x stride (2-way)
  }
}

template <int BYTES>
__global__ void k(unsigned *out, int pat, unsigned zero) {
  __shared__ __align__(16) unsigned char sm[16384 + 4096];
  for (int i = threadIdx.x; i < 16384 + 4096; i += blockDim.x) sm[i] = (unsigned char)(i * 7);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const unsigned base = (unsigned)__cvta_generic_to_shared(sm) + pat_off(pat, lane, BYTES);
  unsigned acc = 0;
  for (int it = 0; it < ITER; ++it) {
    const unsigned b = base + ((it & 1) << 10) + zero;
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      unsigned x, w;
      if (BYTES == 16) {   // volatile: ptxas must not narrow the vector load
        unsigned y, z;
        asm volatile("ld.volatile.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(x), "=r"(y), "=r"(z), "=r"(w) : "r"(b));
      } else {
        asm volatile("ld.volatile.shared.v2.u32 {%0,%1}, [%2];" : "=r"(x), "=r"(w) : "r"(b));
      }
      acc += x + w;     // one IADD3 per load
    }
  }
  if (acc == 0x12345u) out[0] = acc;
}

template <int BYTES>
void run(int sms, unsigned *d, int pat) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int blocks = sms * 4, threads = 256;
  k<BYTES><<<blocks, threads>>>(d, pat, 0u);
  cudaEventRecord(e0);
  k<BYTES><<<blocks, threads>>>(d, pat, 0u);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  int clk_khz; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  double inst = (double)blocks * (threads / 32) * ITER * 16;
  double per_sm_per_clk = inst / (ms * 1e-3) / sms / (clk_khz * 1e3);
  printf("  \"lds%d_pat%d_winst_per_clk\": %.3f,\n", BYTES * 8, pat, per_sm_per_clk);
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned *d; cudaMalloc(&d, 64);
  printf("{\n");
  for (int p = 0; p <= 11; ++p) run<16>(sms, d, p);
  for (int p = 0; p <= 7; ++p) run<8>(sms, d, p);
  printf("  \"sms\": %d\n}\n", sms);
  return 0;
}
