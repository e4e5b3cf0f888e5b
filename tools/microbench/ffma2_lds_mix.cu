// ffma2_lds_mix.cu — ceiling of the FP32 tile kernels' inner-loop instruction
// mix on sm_100a (r02).  One k step of an RA x CB register tile is RA*CB/2
// FFMA2 (a = A value broadcast, b = B pair, accumulator pair) plus, per k,
// CB/4 LDS.128 of B (one k ahead) and, per four k, RA loads of A (LDS.128 of
// four k values, or two LDS.64 when AV = 2).  MODE 0 = FFMA2 only (operands
// already in registers), 1 = + B loads, 2 = + A and B loads (the kernel's
// mix).  Reports the FP32 rate in TFLOP/s at several warps per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ffma2_lds_mix ffma2_lds_mix.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int KSTEPS = 4096;

__device__ __forceinline__ float4 lds4(unsigned a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ float lds1(unsigned a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ float2 lds2(unsigned a) {
  float2 v;
  asm volatile("ld.shared.v2.f32 {%0,%1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a));
  return v;
}

template <int MODE, int RA, int CB, int AV>
__global__ void __launch_bounds__(128) k(float *out, float seed) {
  constexpr int NH = CB / 4;
  __shared__ __align__(16) float sm[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = seed * (float)(i & 7);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  // conflict-free addresses: quarter q of each half reads a different 16-B slot group
  const unsigned base = (unsigned)__cvta_generic_to_shared(sm) + ((lane >> 3) & 1) * 64 + (lane & 3) * 16;
  float2 p[RA][CB / 2];
#pragma unroll
  for (int i = 0; i < RA; ++i)
#pragma unroll
    for (int j = 0; j < CB / 2; ++j) p[i][j] = make_float2(seed * i, seed * j);
  float4 av[RA], bq[NH], bn[NH], aq[RA / 4], an[RA / 4];
  float a1[RA], a1n[RA];
#pragma unroll
  for (int i = 0; i < RA; ++i) a1[i] = a1n[i] = seed * i;
#pragma unroll
  for (int i = 0; i < RA; ++i) av[i] = make_float4(seed, seed * 2, seed * 3, seed * 4);
#pragma unroll
  for (int h = 0; h < NH; ++h) bq[h] = bn[h] = make_float4(seed, seed, seed, seed);
#pragma unroll
  for (int q = 0; q < RA / 4; ++q) aq[q] = an[q] = make_float4(seed, seed, seed, seed);
#pragma unroll 1
  for (int kb = 0; kb < KSTEPS / 4; ++kb) {
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      const unsigned ko = (unsigned)(((kb * 4 + kk) & 63) * 144);
      if (MODE >= 1) {
#pragma unroll
        for (int h = 0; h < NH; ++h) bn[h] = lds4(base + ko + 256 + 128 * h);
      }
      if (MODE == 3) {   // A like B: RA/4 LDS.128 of a transposed copy, one k ahead
#pragma unroll
        for (int q = 0; q < RA / 4; ++q) an[q] = lds4(base + ko + 1024 + 128 * q);
      }
      if (MODE == 4) {   // A one k ahead by RA LDS.32 of M[row][k+1] (row-major, no transposed copy)
#pragma unroll
        for (int i = 0; i < RA; ++i) a1n[i] = lds1(base + ((kb * 4 + kk) & 15) * 4 + i * 144 + 2048);
      }
#pragma unroll
      for (int i = 0; i < RA; ++i) {
        const float a = MODE == 4 ? a1[i] : MODE == 3 ? ((i & 3) == 0 ? aq[i / 4].x : (i & 3) == 1 ? aq[i / 4].y : (i & 3) == 2 ? aq[i / 4].z : aq[i / 4].w)
                        : kk == 0 ? av[i].x : kk == 1 ? av[i].y : kk == 2 ? av[i].z : av[i].w;
#pragma unroll
        for (int h = 0; h < NH; ++h) {
          p[i][2 * h] = __ffma2_rn(make_float2(a, a), make_float2(bq[h].x, bq[h].y), p[i][2 * h]);
          p[i][2 * h + 1] = __ffma2_rn(make_float2(a, a), make_float2(bq[h].z, bq[h].w), p[i][2 * h + 1]);
        }
        if (MODE == 2) {
          const unsigned aa = base + i * 576 + ((kb & 15) << 4);
          if (AV == 4 && kk == 3) av[i] = lds4(aa);
          if (AV == 2 && kk == 1) { const float2 v = lds2(aa); av[i].x = v.x; av[i].y = v.y; }
          if (AV == 2 && kk == 3) { const float2 v = lds2(aa + 8); av[i].z = v.x; av[i].w = v.y; }
        }
      }
      if (MODE >= 1) {
#pragma unroll
        for (int h = 0; h < NH; ++h) bq[h] = bn[h];
      }
      if (MODE == 3) {
#pragma unroll
        for (int q = 0; q < RA / 4; ++q) aq[q] = an[q];
      }
      if (MODE == 4) {
#pragma unroll
        for (int i = 0; i < RA; ++i) a1[i] = a1n[i];
      }
    }
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < RA; ++i)
#pragma unroll
    for (int j = 0; j < CB / 2; ++j) s += p[i][j].x + p[i][j].y;
  if (s == 1.2345f) out[threadIdx.x] = s;
}

template <int MODE, int RA, int CB, int AV>
void run(int sms, float *d, int ctas_per_sm) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int blocks = sms * ctas_per_sm, threads = 128;
  k<MODE, RA, CB, AV><<<blocks, threads>>>(d, 1e-9f);
  cudaEventRecord(e0);
  k<MODE, RA, CB, AV><<<blocks, threads>>>(d, 1e-9f);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, k<MODE, RA, CB, AV>);
  double flops = (double)blocks * threads * KSTEPS * RA * CB * 2;
  printf("  \"mode%d_%dx%d_av%d_warps%d\": {\"tflops\": %.2f, \"regs\": %d},\n", MODE, RA, CB, AV, ctas_per_sm * 4,
         flops / (ms * 1e-3) / 1e12, fa.numRegs);
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float *d; cudaMalloc(&d, 4096);
  printf("{\n");
  for (int c : {2, 3, 4}) {
    run<1, 8, 8, 4>(sms, d, c); run<3, 8, 8, 4>(sms, d, c); run<4, 8, 8, 4>(sms, d, c);
    run<4, 8, 12, 4>(sms, d, c); run<4, 6, 12, 4>(sms, d, c); run<4, 4, 16, 4>(sms, d, c);
  }
  for (int c : {2, 3}) {
    run<3, 8, 16, 4>(sms, d, c); run<4, 8, 16, 4>(sms, d, c); run<4, 12, 12, 4>(sms, d, c); run<4, 6, 16, 4>(sms, d, c);
  }
  printf("  \"sms\": %d\n}\n", sms);
  return 0;
}
