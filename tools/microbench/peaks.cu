// peaks.cu — B200 (sm_100a) pipe/peak microbenchmarks for the batched
// small-matrix update: DFMA, DMMA.8x8x4, FFMA, FFMA2,
// SHFL, LDS.64/128, MOVM, HBM copy.  Prints one JSON object.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o peaks peaks.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

constexpr int ITER = 4096;

__global__ void k_dfma(double *out, double b, double c) {
  double a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < ITER; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void k_dmma(double *out, double av, double bv) {
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = threadIdx.x; c[i][1] = i; }
  double a = av * threadIdx.x, b = bv;
  for (int it = 0; it < ITER / 4; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

// 1 DMMA + 16 DFMA per iteration per warp: do they share the pipe?
__global__ void k_mix(double *out, double av, double bv) {
  double c[4][2], d[8];
#pragma unroll
  for (int i = 0; i < 4; ++i) { c[i][0] = threadIdx.x; c[i][1] = i; }
#pragma unroll
  for (int i = 0; i < 8; ++i) d[i] = i;
  double a = av * threadIdx.x, b = bv;
  for (int it = 0; it < ITER / 4; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
#pragma unroll
      for (int j = 0; j < 8; ++j) d[j] = fma(d[j], b, a);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1];
#pragma unroll
  for (int i = 0; i < 8; ++i) s += d[i];
  if (s == 12345.678) out[0] = s;
}

// The C2 kernel's FP64 instruction mix per warp and update: 16 DMMA.8x8x4
// (4 accumulator chains x 4 k-steps) + 8 DFMA (epilogue).  Upper bound for
// the warp-DMMA n=16 kernel when nothing else stalls.
__global__ void k_mix16_8(double *out, double av, double bv) {
  double c[4][2], d[8];
#pragma unroll
  for (int i = 0; i < 4; ++i) { c[i][0] = threadIdx.x; c[i][1] = i; }
#pragma unroll
  for (int i = 0; i < 8; ++i) d[i] = i;
  double a = av * threadIdx.x, b = bv;
  for (int it = 0; it < ITER / 8; ++it) {
#pragma unroll
    for (int ks = 0; ks < 4; ++ks)
#pragma unroll
      for (int i = 0; i < 4; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
#pragma unroll
    for (int j = 0; j < 8; ++j) d[j] = fma(d[j], b, a);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1];
#pragma unroll
  for (int i = 0; i < 8; ++i) s += d[i];
  if (s == 12345.678) out[0] = s;
}

// The n = 8 kernel's mix per warp and update: 2 DMMA.8x8x4 into ONE
// accumulator (dependent chain) + 2 DFMA (epilogue); DEP = false makes the two
// DMMAs independent (two accumulators), to separate chain latency from the mix.
template <bool DEP>
__global__ void k_mix2_2(double *out, double av, double bv) {
  double c[2][2], d[2];
  c[0][0] = threadIdx.x; c[0][1] = 1; c[1][0] = 2; c[1][1] = 3;
  d[0] = 0.5; d[1] = 0.25;
  double a = av * threadIdx.x, b = bv;
  for (int it = 0; it < ITER / 2; ++it) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c[0][0]), "+d"(c[0][1]) : "d"(a), "d"(b));
    if (DEP)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[0][0]), "+d"(c[0][1]) : "d"(a), "d"(b));
    else
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[1][0]), "+d"(c[1][1]) : "d"(a), "d"(b));
    d[0] = fma(d[0], b, a);
    d[1] = fma(d[1], b, a);
  }
  const double s = c[0][0] + c[0][1] + c[1][0] + c[1][1] + d[0] + d[1];
  if (s == 12345.678) out[0] = s;
}

// The n = 4 thread-per-matrix update's exact DFMA stream (64 product DFMAs in
// k-outer order + 16 epilogue DFMAs per update, whole matrix in registers, no
// memory): the ceiling of the TPM kind's instruction mix.
__global__ void k_tpm4(double *out, int iters) {
  double m[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) m[e] = 1e-3 * (threadIdx.x + e);
  const double c = 0.00005;
  for (int it = 0; it < iters; ++it) {
    double p[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) p[e] = m[e];
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) p[i * 4 + j] = fma(m[i * 4 + k], m[k * 4 + j], p[i * 4 + j]);
#pragma unroll
    for (int e = 0; e < 16; ++e) m[e] = fma(c, p[e], 1.0);
  }
  double s = 0;
#pragma unroll
  for (int e = 0; e < 16; ++e) s += m[e];
  if (s == 12345.678) out[0] = s;
}

__global__ void k_ffma(float *out, float b, float c) {
  float a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < ITER; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = fmaf(a[i], b, c);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i];
  if (s == 12345.678f) out[0] = s;
}

__global__ void k_ffma2(float *out, float b, float c) {
  float2 a[8];
  float2 bb = make_float2(b, b), cc = make_float2(c, c);
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = make_float2(threadIdx.x * 1e-3f + i, i);
  for (int it = 0; it < ITER; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = __ffma2_rn(a[i], bb, cc);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i].x + a[i].y;
  if (s == 12345.678f) out[0] = s;
}

__global__ void k_shfl(int *out) {
  int v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = threadIdx.x + i;
  for (int it = 0; it < ITER / 4; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __shfl_xor_sync(0xffffffffu, v[i], (i + 1) & 31);
  }
  int s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s ^= v[i];
  if (s == 0x7fff1234) out[0] = s;
}

template <int BYTES>
__global__ void k_lds(int *out) {
  extern __shared__ __align__(16) unsigned char sm[];
  for (int i = threadIdx.x; i < 16384; i += blockDim.x) sm[i] = (unsigned char)i;
  __syncthreads();
  int acc = 0;
  unsigned base = (threadIdx.x * BYTES) & 8191;
  for (int it = 0; it < ITER / 4; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      unsigned addr = (base + i * 1024 + (acc & 1) * 0) & 16383;
      if (BYTES == 8) {
        int2 x = *reinterpret_cast<int2 *>(sm + (addr & ~7u));
        acc += x.x ^ x.y;
      } else {
        int4 x = *reinterpret_cast<int4 *>(sm + (addr & ~15u));
        acc += x.x ^ x.y ^ x.z ^ x.w;
      }
    }
    base ^= 64;
  }
  if (acc == 0x7fff1234) out[0] = acc;
}

__global__ void k_movm(int *out) {
  unsigned v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = threadIdx.x * 77u + i;
  for (int it = 0; it < ITER / 4; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %0;" : "+r"(v[i]));
  }
  unsigned s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s ^= v[i];
  if (s == 0x7fff1234u) out[0] = (int)s;
}

__global__ void k_copy(const int4 *__restrict__ a, int4 *__restrict__ b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t st = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += st) b[i] = __ldcs(a + i);
}

template <class F>
static float timeit(F f, int reps = 5) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  f(); CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(e0));
    f();
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  double *dd; float *df; int *di;
  CK(cudaMalloc(&dd, 64)); CK(cudaMalloc(&df, 64)); CK(cudaMalloc(&di, 64));
  const int blocks = sms * 8, threads = 256;
  const double nthr = (double)blocks * threads, nwarp = nthr / 32;
  printf("{\n  \"sms\": %d,\n", sms);
  float ms;
  ms = timeit([&] { k_dfma<<<blocks, threads>>>(dd, 1.0000001, 1e-9); });
  printf("  \"dfma_tflops\": %.3f,\n", nthr * ITER * 8 * 2 / (ms * 1e-3) / 1e12);
  ms = timeit([&] { k_dmma<<<blocks, threads>>>(dd, 1e-3, 1e-3); });
  printf("  \"dmma_tflops\": %.3f,\n", nwarp * (ITER / 4) * 8 * 512.0 / (ms * 1e-3) / 1e12);
  ms = timeit([&] { k_mix<<<blocks, threads>>>(dd, 1e-3, 1e-3); });
  printf("  \"dmma_dfma_mix_tflops\": %.3f,\n",
         (nwarp * (ITER / 4) * 4 * 512.0 + nthr * (ITER / 4) * 4 * 8 * 2.0) / (ms * 1e-3) / 1e12);
  ms = timeit([&] { k_mix16_8<<<blocks, threads>>>(dd, 1e-3, 1e-3); });
  printf("  \"dmma16_dfma8_mix_tflops\": %.3f,\n",
         (nwarp * (ITER / 8) * 16 * 512.0 + nthr * (ITER / 8) * 8 * 2.0) / (ms * 1e-3) / 1e12);
  ms = timeit([&] { k_mix2_2<true><<<blocks, threads>>>(dd, 1e-3, 1e-3); });
  printf("  \"dmma2dep_dfma2_mix_tflops\": %.3f,\n",
         (nwarp * (ITER / 2) * 2 * 512.0 + nthr * (ITER / 2) * 2 * 2.0) / (ms * 1e-3) / 1e12);
  ms = timeit([&] { k_mix2_2<false><<<blocks, threads>>>(dd, 1e-3, 1e-3); });
  printf("  \"dmma2ind_dfma2_mix_tflops\": %.3f,\n",
         (nwarp * (ITER / 2) * 2 * 512.0 + nthr * (ITER / 2) * 2 * 2.0) / (ms * 1e-3) / 1e12);
  {
    // 8 CTAs of 128 per SM, the TPM n = 4 kernel's occupancy
    const int tb = sms * 8, tt = 128, it = ITER / 8;
    ms = timeit([&] { k_tpm4<<<tb, tt>>>(dd, it); });
    printf("  \"tpm4_dfma_stream_tflops\": %.3f,\n", (double)tb * tt * it * 80 * 2 / (ms * 1e-3) / 1e12);
  }
  ms = timeit([&] { k_ffma<<<blocks, threads>>>(df, 1.0000001f, 1e-9f); });
  printf("  \"ffma_tflops\": %.3f,\n", nthr * ITER * 16 * 2 / (ms * 1e-3) / 1e12);
  ms = timeit([&] { k_ffma2<<<blocks, threads>>>(df, 1.0000001f, 1e-9f); });
  printf("  \"ffma2_tflops\": %.3f,\n", nthr * ITER * 8 * 4 / (ms * 1e-3) / 1e12);
  ms = timeit([&] { k_shfl<<<blocks, threads>>>(di); });
  printf("  \"shfl_warp_inst_per_clk_per_sm_at_1965\": %.3f,\n",
         nwarp * (ITER / 4) * 8 / (ms * 1e-3) / sms / 1.965e9);
  ms = timeit([&] { k_lds<8><<<blocks, threads, 16384>>>(di); });
  printf("  \"lds64_bytes_per_clk_per_sm_at_1965\": %.3f,\n",
         nthr * (ITER / 4) * 8 * 8 / (ms * 1e-3) / sms / 1.965e9);
  ms = timeit([&] { k_lds<16><<<blocks, threads, 16384>>>(di); });
  printf("  \"lds128_bytes_per_clk_per_sm_at_1965\": %.3f,\n",
         nthr * (ITER / 4) * 8 * 16 / (ms * 1e-3) / sms / 1.965e9);
  ms = timeit([&] { k_movm<<<blocks, threads>>>(di); });
  printf("  \"movm_warp_inst_per_clk_per_sm_at_1965\": %.3f,\n",
         nwarp * (ITER / 4) * 8 / (ms * 1e-3) / sms / 1.965e9);
  size_t bytes = (size_t)4 << 30;
  int4 *a, *b;
  CK(cudaMalloc(&a, bytes)); CK(cudaMalloc(&b, bytes));
  CK(cudaMemset(a, 1, bytes));
  size_t n = bytes / 16;
  ms = timeit([&] { k_copy<<<sms * 16, 512>>>(a, b, n); });
  printf("  \"hbm_copy_gbs\": %.1f\n}\n", 2.0 * bytes / (ms * 1e-3) / 1e9);
  return 0;
}
