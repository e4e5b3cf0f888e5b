// Throughput of the legacy tensor path on sm_100a for the FP32 kernel's
// instruction: mma.sync m16n8k8 TF32 (SASS HMMA.1688.F32.TF32), 8 independent
// accumulators per warp, many warps per SM.  Prints TFLOP/s (2*1024 flop per mma).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o hmma_tf32 hmma_tf32.cu && ./hmma_tf32
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_hmma(float *out, int iters) {
  unsigned a[4], b[2];
  for (int q = 0; q < 4; ++q) a[q] = __float_as_uint(1.0f + threadIdx.x * 1e-3f + q);
  b[0] = __float_as_uint(0.5f); b[1] = __float_as_uint(0.25f);
  float d[8][4] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(d[j][0]), "+f"(d[j][1]), "+f"(d[j][2]), "+f"(d[j][3])
                   : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  }
  float s = 0;
  for (int j = 0; j < 8; ++j) s += d[j][0] + d[j][1] + d[j][2] + d[j][3];
  if (s == 12345.0f) out[threadIdx.x] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float *o;
  cudaMalloc(&o, 4096);
  const int iters = 4096;
  for (int wpb : {4, 8, 16}) {
    const int blocks = sms * 4;
    k_hmma<<<blocks, 32 * wpb>>>(o, 16);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      k_hmma<<<blocks, 32 * wpb>>>(o, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    const double flops = 2.0 * 1024 * 8 * iters * (double)blocks * wpb;
    printf("{\"warps_per_cta\": %d, \"ctas\": %d, \"ms\": %.4f, \"tf32_mma_sync_tflops\": %.1f, \"per_sm_fma_per_clk_at_1965\": %.1f}\n",
           wpb, blocks, best, flops / best / 1e9, flops / 2 / (best * 1e-3) / sms / 1.965e9);
  }
  return 0;
}
