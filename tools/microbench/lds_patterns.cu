// lds_patterns.cu — shared-memory wavefront cost of LDS.32/64/128 under
// broadcast patterns on sm_100a (used to size the FP32 register tiles).
// Reports warp-instructions per SM-clock (at the reported clock) per pattern;
// 1 / that = wavefronts per instruction.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lds_patterns lds_patterns.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITER = 8192;

template <int BYTES, int PAT>
__global__ void k(int *out, int sel, unsigned zero) {
  __shared__ __align__(16) unsigned char sm[16384];
  for (int i = threadIdx.x; i < 16384; i += blockDim.x) sm[i] = (unsigned char)(i * 7);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  int slot;
  switch (PAT) {
    case 0: slot = lane; break;             // 32 distinct, consecutive
    case 1: slot = lane % 8; break;         // 8 distinct, every quarter reads all 8
    case 2: slot = lane / 4; break;         // 8 distinct, 2 per quarter
    case 3: slot = lane / 8; break;         // 4 distinct, 1 per quarter
    case 4: slot = 0; break;                // broadcast
    case 5: slot = lane % 4; break;         // 4 distinct, all in each quarter
    case 6: slot = (lane % 8) * 2; break;   // 8 distinct at 2x stride
    default: slot = lane / 16; break;       // 2 distinct
  }
  unsigned acc[4] = {0, 0, 0, 0};
  unsigned off = (unsigned)(slot * BYTES);
  for (int it = 0; it < ITER; ++it) {
    const unsigned base = ((it + sel) & 7) * 1024;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      // (acc & zero) == 0 at run time but unknown to the compiler: no hoisting
      const unsigned a = (base + off + u * 256 + (acc[u] & zero)) & 16383u & ~(unsigned)(BYTES - 1);
      if (BYTES == 4) acc[u] += *reinterpret_cast<const unsigned *>(sm + a);
      else if (BYTES == 8) { uint2 v = *reinterpret_cast<const uint2 *>(sm + a); acc[u] += v.x ^ v.y; }
      else { uint4 v = *reinterpret_cast<const uint4 *>(sm + a); acc[u] += v.x ^ v.y ^ v.z ^ v.w; }
    }
  }
  if ((acc[0] ^ acc[1] ^ acc[2] ^ acc[3]) == 0x12345u) out[0] = acc[0];
}

template <int BYTES, int PAT>
void run(int sms, int *d) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int blocks = sms * 4, threads = 512;
  k<BYTES, PAT><<<blocks, threads>>>(d, 0, 0u);
  cudaEventRecord(e0);
  k<BYTES, PAT><<<blocks, threads>>>(d, 1, 0u);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  if (cudaGetLastError() != cudaSuccess) { printf("  \"error\": 1,\n"); return; }
  double inst = (double)blocks * (threads / 32) * ITER * 4;
  double per_sm_per_clk = inst / (ms * 1e-3) / sms / 1.965e9;
  printf("  \"lds%d_pat%d_winst_per_clk\": %.3f,\n", BYTES * 8, PAT, per_sm_per_clk);
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int *d; cudaMalloc(&d, 64);
  printf("{\n");
  run<4, 0>(sms, d); run<4, 1>(sms, d); run<4, 4>(sms, d);
  run<8, 0>(sms, d); run<8, 1>(sms, d); run<8, 2>(sms, d); run<8, 4>(sms, d);
  run<16, 0>(sms, d); run<16, 1>(sms, d); run<16, 2>(sms, d); run<16, 3>(sms, d);
  run<16, 4>(sms, d); run<16, 5>(sms, d); run<16, 6>(sms, d); run<16, 7>(sms, d);
  printf("  \"sms\": %d\n}\n", sms);
  return 0;
}
