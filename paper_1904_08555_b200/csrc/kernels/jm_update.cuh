// jm_update.cuh — device kernels for the batched Eigen-benchmark update
//
//     M <- A + c * (M + M*M),  c = T(0.00005),  repeated `repeat` times
//
// (Listing 4; Listing 5) over
// `batch` independent N x N matrices.  This text is embedded in libjitmat and
// compiled at run time by NVRTC, once per key {N, T, addend} — the B200 analog
// of ClangJIT instantiating `test_jit_sz<type, size>` on first use (Listing 5,
// PAPER.md:397-413; Algorithm 1).  It must stay free of
// #include so NVRTC never touches the file system; jm_plan.h
// is prepended to it when the library embeds the source.
//
// Arithmetic per update: the accumulator starts at M, so
// P = M + M*M costs N^2*N FMAs, then M' = fma(c, P, a_ij) with a_ij = 1 (Ones)
// or [i == j] (Identity) — N^2 (N+1) FMAs per matrix-update in total, the
// algorithmic count.  M*M always reads the pre-update M (Q8 / R8).
#ifndef JM_UPDATE_CUH
#define JM_UPDATE_CUH

namespace jm {

typedef unsigned long long u64;

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ double fmaT(double a, double b, double c) { return __fma_rn(a, b, c); }
__device__ __forceinline__ float fmaT(float a, float b, float c) { return __fmaf_rn(a, b, c); }

__device__ __forceinline__ uint4 ldg_nc16(const void *p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
// 128-bit shared store of two doubles (keeps ptxas from splitting it into two
// 64-bit stores when it cannot prove the swizzled offset is 16-B aligned).
__device__ __forceinline__ void sts_f64x2(void *p, double a, double b) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(p);
  asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(s), "d"(a), "d"(b) : "memory");
}
__device__ __forceinline__ void stg16(void *p, uint4 v) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

// Copy `cnt` packed matrices (MB bytes each) between global memory and a
// shared staging area whose matrices sit SB bytes apart.  Cooperative over NT
// threads; every global access is coalesced.  ALIGNED: the chunk's global start
// is 16-B aligned, so 16-B vectors are used (128-bit LDG/STG).
template <int N, int ES, int SB, int NT, bool ALIGNED>
__device__ __forceinline__ void stage_in(const char *__restrict__ g, char *s, int cnt, int tid) {
  constexpr int MB = N * N * ES;
  if constexpr (ALIGNED && (MB % 16) == 0) {
    constexpr int PPM = MB / 16;
    const int pieces = cnt * PPM;
#pragma unroll 4
    for (int p = tid; p < pieces; p += NT) {
      const int m = p / PPM, q = p - m * PPM;
      *reinterpret_cast<uint4 *>(s + m * SB + q * 16) = ldg_nc16(g + (size_t)p * 16);
    }
  } else if constexpr (ALIGNED && SB == MB) {
    const int bytes = cnt * MB, pieces = bytes >> 4;
#pragma unroll 4
    for (int p = tid; p < pieces; p += NT)
      *reinterpret_cast<uint4 *>(s + p * 16) = ldg_nc16(g + (size_t)p * 16);
    for (int o = pieces * 16 + tid * ES; o < bytes; o += NT * ES) {
      if constexpr (ES == 8) *reinterpret_cast<u64 *>(s + o) = *reinterpret_cast<const u64 *>(g + o);
      else *reinterpret_cast<unsigned *>(s + o) = *reinterpret_cast<const unsigned *>(g + o);
    }
  } else {
    const int elems = cnt * N * N;
    for (int e = tid; e < elems; e += NT) {
      const int m = e / (N * N), q = e - m * (N * N);
      if constexpr (ES == 8)
        *reinterpret_cast<u64 *>(s + m * SB + q * 8) = reinterpret_cast<const u64 *>(g)[e];
      else
        *reinterpret_cast<unsigned *>(s + m * SB + q * 4) = reinterpret_cast<const unsigned *>(g)[e];
    }
  }
}

template <int N, int ES, int SB, int NT, bool ALIGNED>
__device__ __forceinline__ void stage_out(char *__restrict__ g, const char *s, int cnt, int tid) {
  constexpr int MB = N * N * ES;
  if constexpr (ALIGNED && (MB % 16) == 0) {
    constexpr int PPM = MB / 16;
    const int pieces = cnt * PPM;
#pragma unroll 4
    for (int p = tid; p < pieces; p += NT) {
      const int m = p / PPM, q = p - m * PPM;
      stg16(g + (size_t)p * 16, *reinterpret_cast<const uint4 *>(s + m * SB + q * 16));
    }
  } else if constexpr (ALIGNED && SB == MB) {
    const int bytes = cnt * MB, pieces = bytes >> 4;
#pragma unroll 4
    for (int p = tid; p < pieces; p += NT)
      stg16(g + (size_t)p * 16, *reinterpret_cast<const uint4 *>(s + p * 16));
    for (int o = pieces * 16 + tid * ES; o < bytes; o += NT * ES) {
      if constexpr (ES == 8) *reinterpret_cast<u64 *>(g + o) = *reinterpret_cast<const u64 *>(s + o);
      else *reinterpret_cast<unsigned *>(g + o) = *reinterpret_cast<const unsigned *>(s + o);
    }
  } else {
    const int elems = cnt * N * N;
    for (int e = tid; e < elems; e += NT) {
      const int m = e / (N * N), q = e - m * (N * N);
      if constexpr (ES == 8)
        reinterpret_cast<u64 *>(g)[e] = *reinterpret_cast<const u64 *>(s + m * SB + q * 8);
      else
        reinterpret_cast<unsigned *>(g)[e] = *reinterpret_cast<const unsigned *>(s + m * SB + q * 4);
    }
  }
}

// Asynchronous variant of stage_in (cp.async / LDGSTS: global -> shared with no
// register round trip), same layouts; the caller commits and waits.
__device__ __forceinline__ void cp_async16(void *s, const void *g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(s)),
               "l"(g) : "memory");
}
template <int BYTES>
__device__ __forceinline__ void cp_async_small(void *s, const void *g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"((unsigned)__cvta_generic_to_shared(s)),
               "l"(g), "n"(BYTES) : "memory");
}
// zero-filling forms: `src_bytes` (0 or the full size) of the copy come from
// global memory, the rest of the destination is zeroed
__device__ __forceinline__ void cp_async_zfill16(void *s, const void *g, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"((unsigned)__cvta_generic_to_shared(s)),
               "l"(g), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_zfill8(void *s, const void *g, int src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"((unsigned)__cvta_generic_to_shared(s)),
               "l"(g), "r"(src_bytes) : "memory");
}
template <int PENDING>
__device__ __forceinline__ void cp_async_wait_group() { asm volatile("cp.async.wait_group %0;" ::"n"(PENDING) : "memory"); }
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

template <int N, int ES, int SB, int NT, bool ALIGNED>
__device__ __forceinline__ void stage_in_async(const char *__restrict__ g, char *s, int cnt, int tid) {
  constexpr int MB = N * N * ES;
  if constexpr (ALIGNED && (MB % 16) == 0) {
    constexpr int PPM = MB / 16;
    const int pieces = cnt * PPM;
    for (int p = tid; p < pieces; p += NT) {
      const int m = p / PPM, q = p - m * PPM;
      cp_async16(s + m * SB + q * 16, g + (size_t)p * 16);
    }
  } else if constexpr (ALIGNED && SB == MB) {
    const int bytes = cnt * MB, pieces = bytes >> 4;
    for (int p = tid; p < pieces; p += NT) cp_async16(s + p * 16, g + (size_t)p * 16);
    for (int o = pieces * 16 + tid * ES; o < bytes; o += NT * ES) cp_async_small<ES>(s + o, g + o);
  } else {
    const int elems = cnt * N * N;
    for (int e = tid; e < elems; e += NT) {
      const int m = e / (N * N), q = e - m * (N * N);
      cp_async_small<ES>(s + m * SB + q * ES, g + (size_t)e * ES);
    }
  }
}

// ------------------------------------------------ bulk-copy (TMA) primitives
__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(u64 *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(u64 *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(u64 *bar, unsigned parity) {
  unsigned done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!done);
}
// global -> shared, completion counted on `bar` (TMA 1-D bulk copy)
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, u64 *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// shared -> global, tracked by bulk async-groups
__device__ __forceinline__ void bulk_s2g(void *dst, const void *src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
}
// the stage's mbarrier tracks this thread's prior cp.async copies (one
// pending arrival added now, its arrive when they have landed)
__device__ __forceinline__ void cp_async_mbar_arrive(u64 *bar) {
  asm volatile("cp.async.mbarrier.arrive.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read_all() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// make this thread's generic-proxy shared-memory writes visible to the async proxy
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Odd n (a matrix is not a whole number of 16-B pieces; r02): matrix m of a
// chunk, at global byte offset s = (first + m) * MB from the 16-B-aligned
// base, is staged at byte (s & 15) of its SB-byte slot, so the 16-B-aligned
// body of its global range lands 16-B aligned in shared memory and moves by
// 16-B copies; the <= 3 elements before and after the body go one by one.
// Per matrix PPM + 1 work items: body pieces, then one item for head + tail.
template <int N, int ES, int SB, int NT>
__device__ __forceinline__ void stage_in_async_shift(const char *__restrict__ g, long long first, char *s,
                                                     int cnt, int tid) {
  constexpr int MB = N * N * ES, PPM = MB / 16;
  for (int p = tid; p < cnt * (PPM + 1); p += NT) {
    const int m = p / (PPM + 1), q = p - m * (PPM + 1);
    const long long s0 = (first + m) * MB;
    const int sh = (int)(s0 & 15), head = (16 - sh) & 15, nb = (MB - head) >> 4;
    char *d = s + m * SB + sh;
    if (q < nb) {
      cp_async16(d + head + 16 * q, g + s0 + head + 16 * q);
    } else if (q == PPM) {
      for (int o = 0; o < head; o += ES) cp_async_small<ES>(d + o, g + s0 + o);
      for (int o = head + 16 * nb; o < MB; o += ES) cp_async_small<ES>(d + o, g + s0 + o);
    }
  }
}
template <int N, int ES, int SB, int NT>
__device__ __forceinline__ void stage_out_shift(char *__restrict__ g, long long first, const char *s, int cnt,
                                                int tid) {
  constexpr int MB = N * N * ES, PPM = MB / 16;
  for (int p = tid; p < cnt * (PPM + 1); p += NT) {
    const int m = p / (PPM + 1), q = p - m * (PPM + 1);
    const long long s0 = (first + m) * MB;
    const int sh = (int)(s0 & 15), head = (16 - sh) & 15, nb = (MB - head) >> 4;
    const char *d = s + m * SB + sh;
    if (q < nb) {
      stg16(g + s0 + head + 16 * q, *reinterpret_cast<const uint4 *>(d + head + 16 * q));
    } else if (q == PPM) {
      for (int o = 0; o < head; o += ES) *reinterpret_cast<unsigned *>(g + s0 + o) = *reinterpret_cast<const unsigned *>(d + o);
      for (int o = head + 16 * nb; o < MB; o += ES)
        *reinterpret_cast<unsigned *>(g + s0 + o) = *reinterpret_cast<const unsigned *>(d + o);
    }
  }
}

// Chunk scheduler shared by the kernels: a persistent CTA walks chunks of MPC
// matrices (chunk = blockIdx.x, += gridDim.x).  With PF (prefetch) the stage
// area is double-buffered: while chunk i is computed, chunk i+gridDim.x is
// already streaming into the other buffer through cp.async, so the HBM latency
// of the next load hides behind this chunk's updates (matters at small repeat).
//   for (sg.start(); sg.valid(); sg.next()) { sg.acquire(); ...use sg.buf()...; sg.release(); }
// SHIFT (odd n, PF only): each matrix moves by 16-B pieces at byte shift(mi)
// of its slot (stage_in_async_shift / stage_out_shift)
template <int N, int ES, int SB, int NT, int MPC, bool AL, bool PF, bool SHIFT = false>
struct Stager {
  static_assert(!SHIFT || (PF && ES == 4), "shifted staging: the prefetching FP32 stage");
  static constexpr int MB = N * N * ES;
  static constexpr int SZ = rup(MPC * SB, 16);   // one stage buffer
  const char *in;
  char *out;
  char *base;
  long long batch, nchunks, ch;
  int it, tid;
  __device__ __forceinline__ Stager(const void *in_, void *out_, long long batch_, char *base_)
      : in(reinterpret_cast<const char *>(in_)), out(reinterpret_cast<char *>(out_)), base(base_),
        batch(batch_), nchunks((batch_ + MPC - 1) / MPC), ch(blockIdx.x), it(0), tid(threadIdx.x) {}
  __device__ __forceinline__ int count(long long c) const {
    const long long r = batch - c * MPC;
    return (int)(r < MPC ? r : MPC);
  }
  __device__ __forceinline__ void issue(long long c, char *dst) {
    if constexpr (SHIFT) stage_in_async_shift<N, ES, SB, NT>(in, c * MPC, dst, count(c), tid);
    else stage_in_async<N, ES, SB, NT, AL>(in + c * MPC * MB, dst, count(c), tid);
    cp_async_commit();
  }
  // byte offset of matrix mi of the current chunk in its slot (SHIFT)
  __device__ __forceinline__ int shift(int mi) const { return SHIFT ? (int)(((ch * MPC + mi) * MB) & 15) : 0; }
  __device__ __forceinline__ void start() {
    if (PF && ch < nchunks) issue(ch, base);
  }
  __device__ __forceinline__ bool valid() const { return ch < nchunks; }
  __device__ __forceinline__ char *buf() const { return base + (PF ? (it & 1) * SZ : 0); }
  __device__ __forceinline__ int cnt() const { return count(ch); }
  __device__ __forceinline__ void acquire() {
    if constexpr (PF) {
      cp_async_wait_all();
      __syncthreads();   // chunk `ch` visible to all; every thread is done with chunk it-1
      const long long nx = ch + gridDim.x;
      if (nx < nchunks) issue(nx, base + ((it + 1) & 1) * SZ);
    } else {
      stage_in<N, ES, SB, NT, AL>(in + ch * MPC * MB, buf(), cnt(), tid);
      __syncthreads();
    }
  }
  __device__ __forceinline__ void release() {
    __syncthreads();
    if constexpr (SHIFT) stage_out_shift<N, ES, SB, NT>(out, ch * MPC, buf(), cnt(), tid);
    else stage_out<N, ES, SB, NT, AL>(out + ch * MPC * MB, buf(), cnt(), tid);
    if constexpr (!PF) __syncthreads();
  }
  __device__ __forceinline__ void next() {
    ch += gridDim.x;
    ++it;
  }
  __device__ __forceinline__ void finish() {}
  static constexpr int SBM = SB;                                // matrix stride in a stage buffer
  static constexpr int BYTES = (PF ? 2 : 1) * SZ;               // shared memory it occupies
};

// Streaming stager for the HBM-bound (low-repeat) variant, SURVEY.md §8(a)
// a3/a5 "TMA-1D bulk": chunks of K rounds x MPC matrices move through an
// S-stage shared-memory ring of 1-D bulk copies (cp.async.bulk, the TMA
// engine) that complete on one mbarrier per stage; the updated chunk leaves by
// bulk stores straight from the same buffer, so no register ever carries the
// data.  When a matrix is a multiple of 16 B, each matrix is its own copy into
// a slot at the odd-16-B stage stride (stage_stride: the kinds' per-matrix
// shared-memory reads stay bank-conflict free, as in the resident kernel);
// otherwise the chunk is one packed copy.  Warp 0 keeps the ring full: after
// issuing chunk i's stores each of its lanes waits only until its own stores
// have READ their slots, then refills them with chunk i + S, so S - 1 chunk
// loads overlap the compute of chunk i.  A round (what the tiling kinds see
// through buf()/cnt()) is MPC matrices.  The one ragged chunk at the end of
// the batch is staged synchronously with element copies.
// RPB > 0 (row-pitched): each ROW of a matrix is its own bulk copy into the
// slot at a row pitch of RPB bytes, i.e. straight into a kind's padded work
// layout (the rows must be multiples of 16 B); results leave row by row too.
template <int N, int ES, int NT, int MPC, int K, int S, int SLOT = 0, int RPB = 0>
struct Ring {
  static constexpr int MB = N * N * ES;
  static constexpr int ROWB = N * ES;
  static constexpr bool ROWS = RPB > 0;                   // one copy per row
  static_assert(!ROWS || (ROWB % 16 == 0 && RPB % 16 == 0 && RPB >= ROWB), "row-pitched copies of 16-B rows");
  static constexpr bool PER = (MB % 16) == 0;             // one copy per matrix
  // SHF (jm_plan.h ring_shift): matrix m of a full chunk sits at byte
  // shift(m) = (global offset mod 16) of its slot; body by bulk copy, the 8 B
  // outside it by a cp.async whose completion the stage's mbarrier tracks
  static constexpr bool SHF = ring_shift(N, ES, MPC) && !ROWS;
  static constexpr int SBM = ring_sbmr(N, ES, MPC, SLOT);  // matrix slot stride
  static constexpr int RB = MPC * SBM, CHM = K * MPC, CHB = K * RB, GB = CHM * MB;
  static constexpr int TXB = SHF ? CHM * (MB - 8) : GB;   // bytes the bulk copies of a chunk move
  static_assert((SHF || GB % 16 == 0) && CHB % 16 == 0 && TXB % 16 == 0, "bulk copies move multiples of 16 bytes");
  static_assert(S >= 2, "ring of at least two stages");
  static constexpr int BYTES = S * CHB + rup(8 * S, 16);
  const char *in;
  char *out;
  char *base;
  u64 *bar;
  long long batch, nchunks, ch;
  int sub, s, tid;
  unsigned ph;
  __device__ __forceinline__ Ring(const void *in_, void *out_, long long batch_, char *base_)
      : in(reinterpret_cast<const char *>(in_)), out(reinterpret_cast<char *>(out_)), base(base_),
        bar(reinterpret_cast<u64 *>(base_ + S * CHB)), batch(batch_), nchunks((batch_ + CHM - 1) / CHM),
        ch(blockIdx.x), sub(0), s(0), tid(threadIdx.x), ph(0u) {}
  __device__ __forceinline__ bool full(long long c) const { return (c + 1) * CHM <= batch; }
  // warp 0: chunk c -> stage st (the mbarrier's tx count may run ahead of the
  // expect_tx arrival: the phase cannot complete before that arrival)
  __device__ __forceinline__ void issue(long long c, int st) {
    const char *g = in + c * GB;
    char *d = base + st * CHB;
    if constexpr (SHF) {
      // the 8-B pieces first: cp.async.mbarrier.arrive adds a pending arrival
      // BEFORE the expect_tx arrival below, so the phase cannot complete early
      for (int m = tid; m < CHM; m += 32) {
        const int sh = (int)(((c * CHM + m) * MB) & 15), ox = sh ? 0 : MB - 8;
        cp_async_small<8>(d + m * SBM + sh + ox, g + (size_t)m * MB + ox);
        cp_async_mbar_arrive(bar + st);
      }
      __syncwarp();
    }
    if (tid == 0) mbar_expect_tx(bar + st, TXB);
    if constexpr (SHF) {
      for (int m = tid; m < CHM; m += 32) {
        const int sh = (int)(((c * CHM + m) * MB) & 15), ob = sh ? 8 : 0;
        bulk_g2s(d + m * SBM + sh + ob, g + (size_t)m * MB + ob, MB - 8, bar + st);
      }
    } else if constexpr (ROWS) {
      for (int e = tid; e < CHM * N; e += 32) {
        const int m = e / N, r = e - m * N;
        bulk_g2s(d + m * SBM + r * RPB, g + (size_t)e * ROWB, ROWB, bar + st);
      }
    } else if constexpr (PER) {
      for (int m = tid; m < CHM; m += 32) bulk_g2s(d + m * SBM, g + (size_t)m * MB, MB, bar + st);
    } else {
      if (tid == 0) bulk_g2s(d, g, GB, bar + st);
    }
  }
  // warp 0: stage st -> chunk c, one bulk group per issuing lane
  __device__ __forceinline__ void store(long long c, int st) {
    char *g = out + c * GB;
    const char *d = base + st * CHB;
    if constexpr (SHF) {
      for (int m = tid; m < CHM; m += 32) {
        const int sh = (int)(((c * CHM + m) * MB) & 15), ob = sh ? 8 : 0, ox = sh ? 0 : MB - 8;
        bulk_s2g(g + (size_t)m * MB + ob, d + m * SBM + sh + ob, MB - 8);
        *reinterpret_cast<u64 *>(g + (size_t)m * MB + ox) = *reinterpret_cast<const u64 *>(d + m * SBM + sh + ox);
      }
    } else if constexpr (ROWS) {
      for (int e = tid; e < CHM * N; e += 32) {
        const int m = e / N, r = e - m * N;
        bulk_s2g(g + (size_t)e * ROWB, d + m * SBM + r * RPB, ROWB);
      }
    } else if constexpr (PER) {
      for (int m = tid; m < CHM; m += 32) bulk_s2g(g + (size_t)m * MB, d + m * SBM, MB);
    } else {
      if (tid == 0) bulk_s2g(g, d, GB);
    }
    bulk_commit();
  }
  __device__ __forceinline__ void start() {
    if (tid == 0) {
#pragma unroll
      for (int k = 0; k < S; ++k) mbar_init(bar + k, 1);
      fence_mbar_init();
    }
    __syncthreads();
    if (tid < 32) {
#pragma unroll
      for (int k = 0; k < S; ++k) {
        const long long c = ch + (long long)k * gridDim.x;
        if (c < nchunks && full(c)) issue(c, k);
      }
    }
  }
  __device__ __forceinline__ bool valid() const { return ch < nchunks; }
  __device__ __forceinline__ char *buf() const { return base + s * CHB + sub * RB; }
  // byte offset of matrix mi of the current round in its slot (SHF; the
  // ragged last chunk is staged by element copies at offset 0)
  __device__ __forceinline__ int shift(int mi) const {
    return (SHF && full(ch)) ? (int)(((ch * CHM + (long long)sub * MPC + mi) * MB) & 15) : 0;
  }
  __device__ __forceinline__ int cnt() const {
    const long long r = batch - (ch * CHM + (long long)sub * MPC);
    return (int)(r <= 0 ? 0 : (r < MPC ? r : MPC));
  }
  __device__ __forceinline__ void acquire() {
    if (sub != 0) return;
    if (full(ch)) {
      mbar_wait(bar + s, ph);
    } else {   // the ragged last chunk: its stage may still be draining stores
      if (tid < 32) bulk_wait_read_all();
      __syncthreads();
      if constexpr (ROWS) rows_io<true>(const_cast<char *>(in) + ch * GB, base + s * CHB, (int)(batch - ch * CHM));
      else stage_in<N, ES, SBM, NT, false>(in + ch * GB, base + s * CHB, (int)(batch - ch * CHM), tid);
      __syncthreads();
    }
  }
  __device__ __forceinline__ void release() {
    fence_proxy_async();   // this thread's results -> visible to the bulk stores
    __syncthreads();
    if (sub != K - 1) return;
    if (full(ch)) {
      if (tid < 32) {
        store(ch, s);
        const long long nx = ch + (long long)S * gridDim.x;
        if (nx < nchunks && full(nx)) {
#if !JM_RING_NOWAIT_UNSAFE   // (timing experiment only: the refill may overwrite slots a store still reads)
          bulk_wait_read_all();   // this lane's stores have read their slots: refill
#endif
          issue(nx, s);
        }
      }
    } else {
      if constexpr (ROWS) rows_io<false>(out + ch * GB, base + s * CHB, (int)(batch - ch * CHM));
      else stage_out<N, ES, SBM, NT, false>(out + ch * GB, base + s * CHB, (int)(batch - ch * CHM), tid);
    }
  }
  // the ragged chunk, row-pitched: element copies global <-> slot rows
  template <bool IN>
  __device__ __forceinline__ void rows_io(char *g, char *d, int cnt) {
    for (int e = tid; e < cnt * N * N; e += NT) {
      const int m = e / (N * N), q = e - m * (N * N), r = q / N, c = q - r * N;
      char *sp = d + m * SBM + r * RPB + c * ES;
      char *gp = g + (size_t)e * ES;
      if constexpr (ES == 8) {
        if (IN) *reinterpret_cast<u64 *>(sp) = *reinterpret_cast<const u64 *>(gp);
        else *reinterpret_cast<u64 *>(gp) = *reinterpret_cast<const u64 *>(sp);
      } else {
        if (IN) *reinterpret_cast<unsigned *>(sp) = *reinterpret_cast<const unsigned *>(gp);
        else *reinterpret_cast<unsigned *>(gp) = *reinterpret_cast<const unsigned *>(sp);
      }
    }
  }
  __device__ __forceinline__ void next() {
    if (++sub == K) {
      sub = 0;
      ch += gridDim.x;
      if (++s == S) { s = 0; ph ^= 1u; }
    }
  }
  __device__ __forceinline__ void finish() {
    if (tid < 32) bulk_wait_all();
  }
};

template <bool B, class X, class Y> struct Pick { typedef X type; };
template <class X, class Y> struct Pick<false, X, Y> { typedef Y type; };

// ======================================================================
// TPM: thread per matrix.  The whole matrix (and the product) lives in
// registers for all `repeat` updates; fully unrolled for the compile-time N
// (the register analog of Eigen's fixed-size Matrix<T,size,size>).
// ======================================================================
template <int N, class T, Addend A>
__device__ __forceinline__ void tpm_iterate(T (&m)[N * N], int repeat) {
  const T c = T(0.00005);
  for (int r = 0; r < repeat; ++r) {
    T p[N * N];
#pragma unroll
    for (int e = 0; e < N * N; ++e) p[e] = m[e];   // P = M + M*M: accumulators start at M
    // k outermost: consecutive DFMAs share the operand m[i][k] (operand-reuse
    // cache; a DFMA reading three distinct register pairs is register-bank bound)
    // and target independent accumulators; per element the k order is unchanged.
#pragma unroll
    for (int k = 0; k < N; ++k)
#pragma unroll
      for (int i = 0; i < N; ++i)
#pragma unroll
        for (int j = 0; j < N; ++j) p[i * N + j] = fmaT(m[i * N + k], m[k * N + j], p[i * N + j]);
#pragma unroll
    for (int i = 0; i < N; ++i) {
#pragma unroll
      for (int j = 0; j < N; ++j) {
        if (A == Addend::Ones || i == j) m[i * N + j] = fmaT(c, p[i * N + j], T(1));
        else m[i * N + j] = c * p[i * N + j];
      }
    }
  }
}

// FP32 variant: pairs of columns go through FFMA2 (sm_100 packed FP32 FMA):
// half the issue slots of scalar FFMA for the same FMA count.
template <int N, Addend A>
__device__ __forceinline__ void tpm_iterate_f32x2(float (&m)[N * N], int repeat) {
  const float c = float(0.00005);
  constexpr int NH = N / 2;
  for (int r = 0; r < repeat; ++r) {
    float p[N * N];
    float2 p2[N][NH > 0 ? NH : 1];
#pragma unroll
    for (int i = 0; i < N; ++i) {
#pragma unroll
      for (int jj = 0; jj < NH; ++jj) p2[i][jj] = make_float2(m[i * N + 2 * jj], m[i * N + 2 * jj + 1]);
      if constexpr (N % 2) p[i * N + N - 1] = m[i * N + N - 1];
    }
    // k outermost (operand reuse of m[i][k], independent accumulators); per
    // element the k order is unchanged
#pragma unroll
    for (int k = 0; k < N; ++k)
#pragma unroll
      for (int i = 0; i < N; ++i) {
#pragma unroll
        for (int jj = 0; jj < NH; ++jj)
          p2[i][jj] = __ffma2_rn(make_float2(m[i * N + k], m[i * N + k]),
                                 make_float2(m[k * N + 2 * jj], m[k * N + 2 * jj + 1]), p2[i][jj]);
        if constexpr (N % 2)
          p[i * N + N - 1] = fmaT(m[i * N + k], m[k * N + N - 1], p[i * N + N - 1]);
      }
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
      for (int jj = 0; jj < NH; ++jj) {
        p[i * N + 2 * jj] = p2[i][jj].x;
        p[i * N + 2 * jj + 1] = p2[i][jj].y;
      }
#pragma unroll
    for (int i = 0; i < N; ++i) {
#pragma unroll
      for (int j = 0; j < N; ++j) {
        if (A == Addend::Ones || i == j) m[i * N + j] = fmaT(c, p[i * N + j], 1.0f);
        else m[i * N + j] = c * p[i * N + j];
      }
    }
  }
}

// STRM (the low-repeat variant): the same kernel with the double-buffered
// cp.async Stager, so the next chunk streams in while this one is updated.
template <int N, class T, Addend A, bool STRM = false>
__device__ __forceinline__ void run_tpm(const T *__restrict__ in, T *__restrict__ out,
                                        long long batch, int repeat) {
  constexpr int ES = sizeof(T), MB = N * N * ES, SB = stage_stride(N, ES);
  constexpr int NT = TPM_THREADS, MPC = TPM_THREADS;
  extern __shared__ __align__(16) char smem[];
  const int tid = threadIdx.x;
  Stager<N, ES, SB, NT, MPC, true, STRM || prefetch_for(N, ES == 8 ? 1 : 0)> sg(in, out, batch, smem);
  for (sg.start(); sg.valid(); sg.next()) {
    sg.acquire();
    const int cnt = sg.cnt();
    if (tid < cnt) {
      T m[N * N];
      char *mine = sg.buf() + tid * SB;
      if constexpr (MB % 16 == 0) {  // 16-B pieces at an odd 16-B stride: conflict free
#pragma unroll
        for (int q = 0; q < MB / 16; ++q) {
          if constexpr (ES == 8) {
            const double2 v = *reinterpret_cast<const double2 *>(mine + 16 * q);
            m[2 * q] = v.x; m[2 * q + 1] = v.y;
          } else {
            const float4 v = *reinterpret_cast<const float4 *>(mine + 16 * q);
            m[4 * q] = v.x; m[4 * q + 1] = v.y; m[4 * q + 2] = v.z; m[4 * q + 3] = v.w;
          }
        }
      } else {  // odd N: packed, odd element stride: conflict free
#pragma unroll
        for (int e = 0; e < N * N; ++e) m[e] = reinterpret_cast<const T *>(mine)[e];
      }
      if constexpr (ES == 4 && N >= 2) tpm_iterate_f32x2<N, A>(m, repeat);
      else tpm_iterate<N, T, A>(m, repeat);
      if constexpr (MB % 16 == 0) {
#pragma unroll
        for (int q = 0; q < MB / 16; ++q) {
          if constexpr (ES == 8)
            *reinterpret_cast<double2 *>(mine + 16 * q) = make_double2(m[2 * q], m[2 * q + 1]);
          else
            *reinterpret_cast<float4 *>(mine + 16 * q) =
                make_float4(m[4 * q], m[4 * q + 1], m[4 * q + 2], m[4 * q + 3]);
        }
      } else {
#pragma unroll
        for (int e = 0; e < N * N; ++e) reinterpret_cast<T *>(mine)[e] = m[e];
      }
    }
    sg.release();
  }
  sg.finish();
}

// ======================================================================
// TPMS: thread per matrix with the product staged in shared memory (FP64,
// N = 9, 10).  M lives in registers for all updates; P = M + M*M is formed
// one row at a time (N independent accumulator chains, k ascending) and
// parked in the matrix's own staging slot, which is idle between the chunk's
// load and store; once every row of P exists the epilogue M = A + c*P reads
// it back.  Slots of odd 8-B stride (packed, N*N odd) or odd 16-B stride keep
// the lanes' 8-B accesses on distinct banks.
// ======================================================================
template <int N, class T, Addend A>
__device__ __forceinline__ void run_tpms(const T *__restrict__ in, T *__restrict__ out,
                                         long long batch, int repeat) {
  constexpr int ES = sizeof(T), SB = stage_stride(N, ES);
  constexpr int NT = TPM_THREADS, MPC = TPM_THREADS;
  extern __shared__ __align__(16) char smem[];
  const int tid = threadIdx.x;
  const T c = T(0.00005);
  Stager<N, ES, SB, NT, MPC, true, false> sg(in, out, batch, smem);
  for (sg.start(); sg.valid(); sg.next()) {
    sg.acquire();
    if (tid < sg.cnt()) {
      T *slot = reinterpret_cast<T *>(sg.buf() + tid * SB);
      T m[N * N];
#pragma unroll
      for (int e = 0; e < N * N; ++e) m[e] = slot[e];
#pragma unroll 1
      for (int r = 0; r < repeat; ++r) {
#pragma unroll
        for (int i = 0; i < N; ++i) {
          // JM_TPMS_ROWS rows of P live at a time (ptxas would interleave all
          // rows: spills)
          if (i % JM_TPMS_ROWS == 0) asm volatile("" ::: "memory");
          if constexpr (ES == 4) {     // FP32: column pairs through FFMA2
            constexpr int NH = N / 2;
            float2 p2[NH > 0 ? NH : 1];
            float pl = 0.0f;
#pragma unroll
            for (int jj = 0; jj < NH; ++jj) p2[jj] = make_float2(m[i * N + 2 * jj], m[i * N + 2 * jj + 1]);
            if constexpr (N % 2) pl = m[i * N + N - 1];
#pragma unroll
            for (int k = 0; k < N; ++k) {
              const float a = m[i * N + k];
#pragma unroll
              for (int jj = 0; jj < NH; ++jj)
                p2[jj] = __ffma2_rn(make_float2(a, a), make_float2(m[k * N + 2 * jj], m[k * N + 2 * jj + 1]), p2[jj]);
              if constexpr (N % 2) pl = fmaT(a, m[k * N + N - 1], pl);
            }
#pragma unroll
            for (int jj = 0; jj < NH; ++jj) {
              slot[i * N + 2 * jj] = p2[jj].x;
              slot[i * N + 2 * jj + 1] = p2[jj].y;
            }
            if constexpr (N % 2) slot[i * N + N - 1] = pl;
          } else {
            T p[N];
#pragma unroll
            for (int j = 0; j < N; ++j) p[j] = m[i * N + j];      // accumulators start at M
#pragma unroll
            for (int k = 0; k < N; ++k)
#pragma unroll
              for (int j = 0; j < N; ++j) p[j] = fmaT(m[i * N + k], m[k * N + j], p[j]);
#pragma unroll
            for (int j = 0; j < N; ++j) slot[i * N + j] = p[j];
          }
        }
#pragma unroll
        for (int i = 0; i < N; ++i)
#pragma unroll
          for (int j = 0; j < N; ++j) {
            const T pv = slot[i * N + j];
            m[i * N + j] = (A == Addend::Ones || i == j) ? fmaT(c, pv, T(1)) : c * pv;
          }
      }
#pragma unroll
      for (int e = 0; e < N * N; ++e) slot[e] = m[e];
    }
    sg.release();
  }
  sg.finish();
}

// ======================================================================
// DMMA: FP64 tensor cores (mma.sync.m8n8k4.f64 -> SASS DMMA.8x8x4).
//
// M is padded to NP = 8*T8 and held in registers as DMMA accumulator
// fragments: lane (g = lane/4, t = lane%4) holds M[8I+g][8J+2t+s], s = 0,1.
// k-permutation: the k-step (J, s) sums over k in {8J + 2t + s : t = 0..3}.
// With that grouping the A fragment A[g][t] = M[8I+g][8J+2t+s] is exactly the
// lane's own accumulator element s of tile (I, J) — no data movement.  The B
// fragment B[t][g] = M[8J+2t+s][8J'+g] is the transpose-side read; it goes
// through a shared-memory copy of M that each update republishes, in an
// XOR-swizzled layout that makes both the 128-bit publish stores and the 64-bit
// fragment loads bank-conflict free.
// W warps share one matrix (each owns RT row tiles); W == 1 for N <= 32.
// ======================================================================
__device__ __forceinline__ void dmma884(double &d0, double &d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}
// D = A*B + C with D != C: the first k-step reads the accumulator init (M)
// from the A-operand registers directly, so P needs no separate copy of M.
__device__ __forceinline__ void dmma884_c(double &d0, double &d1, double a, double b, double c0,
                                          double c1) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};"
      : "=d"(d0), "=d"(d1)
      : "d"(a), "d"(b), "d"(c0), "d"(c1));
}

// Scratch layout: 16-B chunk `cc` of row `r` lives at byte
//   (r * RSC + (cc ^ ((r & 6) ^ ((r & 1) << 2)))) * 16
// (run_dmma precomputes this as lane constants + immediates: bofs / pofs).

template <int N, Addend A, int W, bool STRM>
__device__ __forceinline__ void run_dmma(const double *__restrict__ in, double *__restrict__ out,
                                         long long batch, int repeat) {
  constexpr int T8 = dmma_t8(N), RT = dmma_rt(N, STRM), RSC = dmma_rsc(N), SCR = dmma_scr(N);
  constexpr int ES = 8, MB = N * N * 8, SB = stage_stride(N, 8);
  constexpr int WPC = (W == 1) ? DMMA_WPC : W;
  constexpr int NT = 32 * WPC;
  constexpr int MPC = (W == 1) ? DMMA_WPC : 1;
  constexpr bool AL = ((MPC * MB) % 16) == 0;
  static_assert(RT * W >= T8 && RT * (W - 1) < T8, "row tiles must cover the matrix");
  // RAG: the last warp owns fewer row tiles (T8 = 7 as 4 + 3); its phantom
  // tiles are skipped by warp-uniform branches
  constexpr bool RAG = RT * W != T8;
  constexpr bool PF = prefetch_for(N, 1);
  typedef typename Pick<STRM, Ring<N, ES, NT, MPC, ring_kr(N, ES, MPC), JM_RING_S, dmma_slot(N)>,
                        Stager<N, ES, SB, NT, MPC, AL, PF>>::type Stg;
  // streaming, even n: the matrix's ring slot (widened to the publish buffer
  // when needed, dmma_slot) doubles as its (first) publish buffer once M is in
  // the accumulators (plan_stream)
  constexpr bool INPL = STRM && dmma_inplace(N);
  // thin border (n = 8K + BR, BR <= JM_DMMA_BORDER_MAX, whole matrix per warp):
  // the last row / column tile holds only BR real rows / columns, so its
  // 2K + 1 tiles are not sent through DMMA (7/8 of that work would be
  // padding); their entries are dot products formed with DFMA from the lanes'
  // own accumulators and the published M, reduced across the warp by shuffles.
  // Measured (r01_dmma_border_sweep): FP64 pipe at R = 100, n = 17 0.41 ->
  // 0.54, 25 0.53 -> 0.67, 33 0.59 -> 0.73, 18 0.40 -> 0.43, 26 0.51 -> 0.56,
  // 34 0.58 -> 0.64; at n = 9 / 10 (one main tile) the shuffles cost what the
  // DMMAs save (0.23 -> 0.23 / 0.19), so those keep the padded tiles.
  // (Only for whole-matrix warps: a several-warp version, where the warp
  // owning the border row tile forms the row border, measured slower — n = 41
  // 0.63 -> 0.48, 57 0.68 -> 0.53 of the pipe, profiles/r01_dmma_border_multiwarp.jsonl —
  // and was removed in r02.)
  constexpr int BR = N - 8 * (T8 - 1);
  constexpr bool BORD = (W == 1) && (N > JM_DMMA_BORDER_MIN) && (BR <= JM_DMMA_BORDER_MAX);
  constexpr int KTOP = BORD ? T8 - 1 : T8;   // global row tiles through DMMA
  constexpr int KN = BORD ? T8 - 1 : T8;     // column tiles through DMMA
  // k-compaction (jm_plan.h JM_DMMA_KCOMPACT): the last k tile's BR <= 4 real
  // k go through ONE k-step, k_t = 8(T8-1) + t.  Its A fragment M[8I+g][8K+t]
  // sits in slot t&1 of lane (g, t>>1): two shuffles per row tile.  Its B
  // fragment is the plain read of row 8K+t of the published M.
  constexpr bool CMP = JM_DMMA_KCOMPACT && T8 >= 2 && BR >= 2 && BR <= 4;
  extern __shared__ __align__(16) char smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int mi = (W == 1) ? warp : 0;        // matrix slot in the chunk
  const int wr = (W == 1) ? 0 : warp;        // this warp's rank within the matrix
  // ONE (r02, streaming CTA kernels): a single publish buffer and one more
  // CTA barrier per update instead of two alternating buffers — at the low
  // repeat counts this kernel runs (one update at R = 1) the second buffer
  // was mostly idle shared memory (jm_plan.h JM_DMMA_STREAM_1BUF)
  constexpr bool ONE = STRM && W > 1 && !INPL && dmma_stream_1buf(N);
  char *scr = smem + Stg::BYTES + ((W == 1 && !INPL) ? warp * SCR : 0);
  const double c = 0.00005;
  // Swizzled-scratch offsets factored into a few lane constants plus
  // compile-time immediates (chunk c ^ f only touches c's low 3 bits, and the
  // row swizzle f depends on the row mod 8 alone):
  //   B fragment, k-step (J,s), column tile J2:  bofs[s][J2&1] + (8J*RSC + 8(J2>>1))*16
  //   publish, own row tile I, column tile J:    pofs[J&1] + (8I*RSC + 8(J>>1))*16
  // so ptxas keeps 6 registers of addresses instead of one per (J, s, J2).
  const int gh = g >> 1, gl = g & 1, fg = (g & 6) ^ ((g & 1) << 2);
  int bofs[2][2], pofs[2];
#pragma unroll
  for (int s = 0; s < 2; ++s)
#pragma unroll
    for (int j1 = 0; j1 < 2; ++j1)
      bofs[s][j1] = ((2 * t + s) * RSC + ((j1 * 4 + gh) ^ (2 * t ^ (s << 2)))) * 16 + 8 * gl;
#pragma unroll
  for (int j1 = 0; j1 < 2; ++j1) pofs[j1] = ((8 * wr * RT + g) * RSC + ((j1 * 4 + t) ^ fg)) * 16;
  // border (BORD): column pair (8K, 8K+1) of row 8J + 2t + s -> colofs[s] + 8J*RSC*16
  // (the pair (8K+2, 8K+3) 16 B further);
  // element (8K + g', 8I + g) -> rowofs + (g'*RSC + 4*(I ^ (g' & 1)) + (g' & 2))*16
  int colofs[2] = {0, 0}, rowofs = 0;
  if constexpr (BORD) {
#pragma unroll
    for (int s = 0; s < 2; ++s) colofs[s] = ((2 * t + s) * RSC + ((4 * (T8 - 1)) ^ (2 * t ^ (s << 2)))) * 16;
    rowofs = (8 * (T8 - 1) * RSC + gh) * 16 + 8 * gl;
  }
  // compacted k-step (CMP): B fragment M[8K + t][8J2 + g] -> cofs[J2&1] + (8K*RSC + 8(J2>>1))*16
  // (row 8K + t has swizzle (t & 2) ^ ((t & 1) << 2)); A fragment source lane (g, t >> 1)
  int cofs[2] = {0, 0};
  const int csrc = (lane & ~3) | (t >> 1);
  if constexpr (CMP) {
#pragma unroll
    for (int j1 = 0; j1 < 2; ++j1) cofs[j1] = (t * RSC + ((j1 * 4 + gh) ^ ((t & 2) ^ ((t & 1) << 2)))) * 16 + 8 * gl;
  }

  Stg sg(in, out, batch, smem);
  for (sg.start(); sg.valid(); sg.next()) {
    sg.acquire();
    char *stage = sg.buf();
    const int cnt = sg.cnt();
    if (mi < cnt) {
      double *sm = reinterpret_cast<double *>(stage + mi * Stg::SBM + sg.shift(mi));   // (odd n: Ring SHF)
      double acc[RT][T8][2];
      if constexpr (N % 2 == 0) {
        // even n: the lane's pair (8J+2t, 8J+2t+1) is one 16-B load; for n a
        // multiple of 16 (rows 2^k * 128 B apart) the odd-g lanes take the
        // column tiles of a pair in the other order, so a quarter-warp's two
        // rows land in different bank slots (the element loads were 8-way
        // conflicted: half the time of a streaming update at n = 64)
        constexpr bool SWZ = (N % 16 == 0) && (T8 % 2 == 0);
        const int odd = SWZ ? (g & 1) : 0;
#pragma unroll
        for (int I = 0; I < RT; ++I) {
          const int row = 8 * (wr * RT + I) + g;
#pragma unroll
          for (int J = 0; J < T8; ++J) {
            const int Jr = J ^ odd;                 // the column tile this lane loads now
            double2 v = make_double2(0.0, 0.0);
            if (row < N && 8 * Jr + 2 * t < N) v = *reinterpret_cast<const double2 *>(sm + row * N + 8 * Jr + 2 * t);
            if (SWZ && odd) { acc[I][J ^ 1][0] = v.x; acc[I][J ^ 1][1] = v.y; }
            else { acc[I][J][0] = v.x; acc[I][J][1] = v.y; }
          }
        }
      } else {
#pragma unroll
        for (int I = 0; I < RT; ++I)
#pragma unroll
          for (int J = 0; J < T8; ++J)
#pragma unroll
            for (int s = 0; s < 2; ++s) {
              const int row = 8 * (wr * RT + I) + g, col = 8 * J + 2 * t + s;
              acc[I][J][s] = (row < N && col < N) ? sm[row * N + col] : 0.0;
            }
      }
      if constexpr (INPL) {                  // every warp has read M before the slot is reused
        if constexpr (W == 1) __syncwarp(); else __syncthreads();
      }
      for (int r = 0; r < repeat; ++r) {
        char *sb = INPL ? ((W > 1 && (r & 1)) ? scr : reinterpret_cast<char *>(sm))
                        : scr + ((W > 1 && !ONE) ? (r & 1) * SCR : 0);
        if constexpr (ONE) {           // every B-fragment read of update r-1 done before this publish
          if (r > 0) __syncthreads();
        }
        // publish M (own rows) for the B-fragment reads
#pragma unroll
        for (int I = 0; I < RT; ++I) {
          if (RAG && wr * RT + I >= T8) continue;
#pragma unroll
          for (int J = 0; J < T8; ++J)
            sts_f64x2(sb + pofs[J & 1] + (8 * I * RSC + 8 * (J >> 1)) * 16, acc[I][J][0], acc[I][J][1]);
        }
        if constexpr (W == 1) __syncwarp(); else __syncthreads();
        double p[RT][T8][2];
        if constexpr (BORD) {
          constexpr int K = T8 - 1;
          // column border P[8I+g][8K+c] (c < BR), this warp's row tiles: lane
          // (g,t) sums its own k = 8J+2t+s terms, then the 4 lanes of a row add up
          constexpr int NCC = BR <= 2 ? 2 : 4;   // border columns formed (the rest of a chunk is padding)
          double cs[RT][NCC];
#pragma unroll
          for (int I = 0; I < RT; ++I)
#pragma unroll
            for (int cc = 0; cc < NCC; ++cc) cs[I][cc] = 0.0;
#pragma unroll
          for (int J = 0; J < T8; ++J)
#pragma unroll
            for (int s = 0; s < 2; ++s) {
              if (8 * J + s >= N) continue;
              const char *q = sb + colofs[s] + 8 * J * RSC * 16;
              double v[NCC];
              if constexpr (BR == 1) {
                v[0] = *reinterpret_cast<const double *>(q);
                v[1] = 0.0;
              } else {
#pragma unroll
                for (int h = 0; h < NCC / 2; ++h) {   // chunk 4K + h sits 16 B after chunk 4K (XOR touches bits 1, 2)
                  const double2 w = *reinterpret_cast<const double2 *>(q + 16 * h);
                  v[2 * h] = w.x; v[2 * h + 1] = w.y;
                }
              }
#pragma unroll
              for (int I = 0; I < RT; ++I)
#pragma unroll
                for (int cc = 0; cc < NCC; ++cc)
                  if (cc < BR) cs[I][cc] = fmaT(acc[I][J][s], v[cc], cs[I][cc]);
            }
#pragma unroll
          for (int I = 0; I < RT; ++I) {
            if constexpr (NCC == 2) {
#pragma unroll
              for (int cc = 0; cc < 2; ++cc) {
                double v = cs[I][cc];
                if (cc < BR) {
                  v += __shfl_xor_sync(0xffffffffu, v, 1);
                  v += __shfl_xor_sync(0xffffffffu, v, 2);
                }
                p[I][K][cc] = (cc < BR && t == 0) ? acc[I][K][cc] + v : 0.0;
              }
            } else {
              // reduce-scatter over the 4 lanes of a row: even t keeps columns
              // (0, 1), odd t (2, 3); then the pair adds across t ^ 2
              const bool od = t & 1;
              const double r0 = __shfl_xor_sync(0xffffffffu, od ? cs[I][0] : cs[I][2], 1);
              const double r1 = __shfl_xor_sync(0xffffffffu, od ? cs[I][1] : cs[I][3], 1);
              double k0 = (od ? cs[I][2] : cs[I][0]) + r0, k1 = (od ? cs[I][3] : cs[I][1]) + r1;
              k0 += __shfl_xor_sync(0xffffffffu, k0, 2);
              k1 += __shfl_xor_sync(0xffffffffu, k1, 2);
              p[I][K][0] = (t < 2 && 2 * t < BR) ? acc[I][K][0] + k0 : 0.0;
              p[I][K][1] = (t < 2 && 2 * t + 1 < BR) ? acc[I][K][1] + k1 : 0.0;
            }
          }
          // row border P[8K+g'][8J+2t+s] (g' < BR), column tiles J < K: lane
          // (g,t) sums the k = 8I+g terms from its accumulators, then the 8
          // lanes of a column add up
          constexpr int IK = K;              // (whole matrix per warp: RT = T8)
          auto finish_row = [&](int J, int s, const double (&rsv)[BR]) {
            double mine = 0.0;
            if constexpr (BR == 1) {
              double v = rsv[0];
              v += __shfl_xor_sync(0xffffffffu, v, 4);
              v += __shfl_xor_sync(0xffffffffu, v, 8);
              v += __shfl_xor_sync(0xffffffffu, v, 16);
              mine = v;
            } else {
              // reduce-scatter over the 8 lanes of a column (g): g bit 0 picks
              // rows {0, 2} / {1, 3}, g bit 1 the row of the pair, g bit 2 adds
              const bool g0 = g & 1, g1 = (g >> 1) & 1;
              const double v2 = BR > 2 ? rsv[BR > 2 ? 2 : 0] : 0.0, v3 = BR > 3 ? rsv[BR > 3 ? 3 : 0] : 0.0;
              const double r0 = __shfl_xor_sync(0xffffffffu, g0 ? rsv[0] : rsv[1], 4);
              double w0 = (g0 ? rsv[1] : rsv[0]) + r0, w1 = 0.0;
              if constexpr (BR > 2) {
                const double r1 = __shfl_xor_sync(0xffffffffu, g0 ? v2 : v3, 4);
                w1 = (g0 ? v3 : v2) + r1;
                const double r = __shfl_xor_sync(0xffffffffu, g1 ? w0 : w1, 8);
                mine = (g1 ? w1 : w0) + r;
              } else {
                mine = w0 + __shfl_xor_sync(0xffffffffu, w0, 8);   // (g1 = 1 lanes hold rows >= 2: unused)
              }
              mine += __shfl_xor_sync(0xffffffffu, mine, 16);
            }
            p[IK][J][s] = (g < BR) ? acc[IK][J][s] + mine : 0.0;
          };
          if constexpr (BR * K <= 8) {       // I outer: each border-row value loaded once
            double rs[BR][K > 0 ? K : 1][2];
#pragma unroll
            for (int q = 0; q < BR; ++q)
#pragma unroll
              for (int J = 0; J < K; ++J) rs[q][J][0] = rs[q][J][1] = 0.0;
#pragma unroll
            for (int I = 0; I < T8; ++I) {
              double mr[BR];
#pragma unroll
              for (int q = 0; q < BR; ++q)
                mr[q] = *reinterpret_cast<const double *>(sb + rowofs + (q * RSC + 4 * (I ^ (q & 1)) + (q & 2)) * 16);
#pragma unroll
              for (int q = 0; q < BR; ++q)
#pragma unroll
                for (int J = 0; J < K; ++J)
#pragma unroll
                  for (int s = 0; s < 2; ++s) rs[q][J][s] = fmaT(mr[q], acc[I][J][s], rs[q][J][s]);
            }
#pragma unroll
            for (int J = 0; J < K; ++J)
#pragma unroll
              for (int s = 0; s < 2; ++s) {
                double rsv[BR];
#pragma unroll
                for (int q = 0; q < BR; ++q) rsv[q] = rs[q][J][s];
                finish_row(J, s, rsv);
              }
          } else {                           // J outer (fewer live sums; the row values are reloaded per J)
#pragma unroll
            for (int J = 0; J < K; ++J) {
              double rs[2][BR];
#pragma unroll
              for (int q = 0; q < BR; ++q) rs[0][q] = rs[1][q] = 0.0;
#pragma unroll
              for (int I = 0; I < T8; ++I)
#pragma unroll
                for (int q = 0; q < BR; ++q) {
                  const double mr =
                      *reinterpret_cast<const double *>(sb + rowofs + (q * RSC + 4 * (I ^ (q & 1)) + (q & 2)) * 16);
                  rs[0][q] = fmaT(mr, acc[I][J][0], rs[0][q]);
                  rs[1][q] = fmaT(mr, acc[I][J][1], rs[1][q]);
                }
              finish_row(J, 0, rs[0]);
              finish_row(J, 1, rs[1]);
            }
          }
        }
#pragma unroll
        for (int J = 0; J < T8; ++J) {
#pragma unroll
          for (int s = 0; s < 2; ++s) {
            if (8 * J + s >= N) continue;   // every k of this k-step is padding: skip (compile time)
            const bool cmp = CMP && J == T8 - 1;   // the compacted last k-step (compile time)
            if (cmp && s == 1) continue;
            double b[KN];
#pragma unroll
            for (int J2 = 0; J2 < KN; ++J2)
              b[J2] = *reinterpret_cast<const double *>(sb + (cmp ? cofs[J2 & 1] : bofs[s][J2 & 1]) +
                                                        (8 * J * RSC + 8 * (J2 >> 1)) * 16);
#pragma unroll
            for (int I = 0; I < RT; ++I) {
              if ((RAG || BORD) && wr * RT + I >= KTOP) continue;   // border / phantom row tile
              double a = acc[I][J][s];
              if (cmp) {
                const double a0 = __shfl_sync(0xffffffffu, acc[I][J][0], csrc);
                const double a1 = __shfl_sync(0xffffffffu, acc[I][J][1], csrc);
                a = (t & 1) ? a1 : a0;
              }
#pragma unroll
              for (int J2 = 0; J2 < KN; ++J2) {
                if (J == 0 && s == 0)   // P = M + (first k-step): accumulator init is M itself
                  dmma884_c(p[I][J2][0], p[I][J2][1], a, b[J2], acc[I][J2][0], acc[I][J2][1]);
                else
                  dmma884(p[I][J2][0], p[I][J2][1], a, b[J2]);
              }
            }
          }
        }
        // M' = A + c * P  (padding stays exactly zero)
#pragma unroll
        for (int I = 0; I < RT; ++I)
#pragma unroll
          for (int J = 0; J < T8; ++J)
#pragma unroll
            for (int s = 0; s < 2; ++s) {
              const int row = 8 * (wr * RT + I) + g, col = 8 * J + 2 * t + s;
              const double a = (A == Addend::Ones || row == col) ? 1.0 : 0.0;
              double v = fmaT(c, p[I][J][s], a);
              if constexpr (N % 8 != 0 || RAG) v = (row < N && col < N) ? v : 0.0;
              acc[I][J][s] = v;
            }
        if constexpr (W == 1) __syncwarp();
      }
      if constexpr (INPL && W > 1) __syncthreads();   // last B-fragment reads of the slot done
      if constexpr (N % 2 == 0) {              // the same 16-B pattern back
        constexpr bool SWZ = (N % 16 == 0) && (T8 % 2 == 0);
        const int odd = SWZ ? (g & 1) : 0;
#pragma unroll
        for (int I = 0; I < RT; ++I) {
          const int row = 8 * (wr * RT + I) + g;
#pragma unroll
          for (int J = 0; J < T8; ++J) {
            const int Jr = J ^ odd;
            const double2 v = (SWZ && odd) ? make_double2(acc[I][J ^ 1][0], acc[I][J ^ 1][1])
                                           : make_double2(acc[I][J][0], acc[I][J][1]);
            if (row < N && 8 * Jr + 2 * t < N) *reinterpret_cast<double2 *>(sm + row * N + 8 * Jr + 2 * t) = v;
          }
        }
      } else {
#pragma unroll
        for (int I = 0; I < RT; ++I)
#pragma unroll
          for (int J = 0; J < T8; ++J)
#pragma unroll
            for (int s = 0; s < 2; ++s) {
              const int row = 8 * (wr * RT + I) + g, col = 8 * J + 2 * t + s;
              if (row < N && col < N) sm[row * N + col] = acc[I][J][s];
            }
      }
    }
    sg.release();
  }
  sg.finish();
}

// ======================================================================
// F32P: FP32 row panels (9 <= N <= 32).  Each of the G threads of a matrix
// owns RP = 4 FULL rows of M in registers, so the A operand of P = M + M*M
// (M[i][k] for its rows) is local; the B operand (row k of M) is a
// shared-memory broadcast: the G threads of a matrix read the same 16-B
// chunks.  Per update a thread issues 4*N/2 FFMA2 per k against N/4 LDS.128.
// Rows live in a double-buffered shared copy (one __syncwarp per update):
// update r reads buffer r&1 and writes its new rows into buffer (r&1)^1.
// 16-B chunk q of row r is stored at chunk q ^ ((r >> 2) & (NCS-1)), so the
// 4 (or 8) threads of a matrix publishing row r0+i hit distinct bank groups.
// For N > 16 the accumulators are formed in two column halves (the 4 full
// rows of the A operand stay in registers for both).
// ======================================================================
template <int NCS>
__device__ __forceinline__ int f32p_off(int row, int q) {
  return (row * NCS + (q ^ ((row >> 2) & (NCS - 1)))) * 16;
}

template <int N, Addend A, bool STRM>
__device__ __forceinline__ void run_f32p(const float *__restrict__ in, float *__restrict__ out,
                                         long long batch, int repeat) {
  constexpr int RP = f32p_rp(N), G = f32p_g(N), MPW = f32p_mpw(N), NCR = f32p_ncr(N);
  static_assert(RP <= F32P_RP_MAX, "at most 4 resident rows per thread");
  constexpr int NCS = f32p_ncs(N), HALVES = f32p_halves(N), MBUF = f32p_mbuf(N);
  constexpr int NC = 4 * NCR;                          // computed columns (16-B padded)
  constexpr int QH = cdiv(NCR, HALVES);                     // chunks per column group
  constexpr int ES = 4, MB = N * N * 4;
  // resident: the staged matrix's slot (f32p_slot bytes) doubles as the first
  // of its two row buffers once the rows sit in registers, so only the second
  // buffer needs its own area (f32p_inplace); streaming: two own buffers
  // (streaming: the same with ring slots widened to a row buffer, f32p_ring_inplace)
  constexpr bool INPL = STRM ? f32p_ring_inplace(N) : f32p_inplace(N);
  constexpr int SB = INPL ? f32p_slot(N) : stage_stride(N, 4);
  constexpr int NT = 32 * F32P_WPC, MPC = F32P_WPC * MPW;
  constexpr bool AL = ((MPC * MB) % 16) == 0;
  static_assert(G * RP >= N, "row panels must cover the matrix");
  constexpr bool PF = prefetch_for(N, 0);
  typedef typename Pick<STRM, Ring<N, ES, NT, MPC, ring_kr(N, ES, MPC), JM_RING_S, INPL ? f32p_slot(N) : 0>,
                        Stager<N, ES, SB, NT, MPC, AL, PF>>::type Stg;
  extern __shared__ __align__(16) char smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int mw = lane / G, tg = lane - mw * G;
  const int mi = warp * MPW + mw;                      // matrix slot in the chunk
  const int r0 = tg * RP;
  constexpr int PSTR = INPL ? MBUF : f32p_pstr(N);   // per-matrix buffer stride
  char *bufs = smem + Stg::BYTES + mi * PSTR;
  const float c = float(0.00005);

  Stg sg(in, out, batch, smem);
  for (sg.start(); sg.valid(); sg.next()) {
    sg.acquire();
    char *stage = sg.buf();
    const int cnt = sg.cnt();
    // every lane runs the loop (a warp holds several matrices and syncs as one);
    // slots past the batch end compute on zeros and are never written back
    const bool live = mi < cnt;
    float *sm = reinterpret_cast<float *>(stage + mi * Stg::SBM);
    // the two row buffers: b0 (the slot itself when INPL) and b1
    char *b0 = INPL ? reinterpret_cast<char *>(sm) : bufs;
    char *b1 = INPL ? bufs : bufs + MBUF;
    float m[RP][NC];
    // VCP (own row buffers, rows of whole 16-B chunks): the warp copies its
    // matrices' packed slots into their first row buffers chunk by chunk (lane
    // = consecutive chunks: both sides bank-conflict free), then each thread
    // reads its rows back with LDS.128 in the publish pattern.  r02: the
    // per-element reads of the packed slot put a matrix's 4 threads (rows
    // 256 B apart) on one bank (60 % of the ring kernel's wavefronts conflicted
    // at n = 16, R = 1; profiles/r02_ncu_baseline_f32.md)
    constexpr bool VCP = !INPL && (N % 4 == 0);
    constexpr int CPM = N * NCR;                  // 16-B chunks per matrix
    if constexpr (VCP) {
#pragma unroll 4
      for (int e = lane; e < MPW * CPM; e += 32) {
        const int ml = e / CPM, cc = e - ml * CPM, row = cc / NCR, q = cc - row * NCR, ms = warp * MPW + ml;
        const float4 v = ms < cnt ? *reinterpret_cast<const float4 *>(stage + ms * Stg::SBM + cc * 16)
                                  : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        *reinterpret_cast<float4 *>(smem + Stg::BYTES + ms * PSTR + f32p_off<NCS>(row, q)) = v;
      }
      __syncwarp();
#pragma unroll
      for (int i = 0; i < RP; ++i)
#pragma unroll
        for (int q = 0; q < NCR; ++q) {
          float4 v = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
          if (r0 + i < N) v = *reinterpret_cast<const float4 *>(b0 + f32p_off<NCS>(r0 + i, q));
          m[i][4 * q] = v.x; m[i][4 * q + 1] = v.y; m[i][4 * q + 2] = v.z; m[i][4 * q + 3] = v.w;
        }
#pragma unroll
      for (int i = 0; i < RP; ++i)
#pragma unroll
        for (int j = 4 * NCR; j < NC; ++j) m[i][j] = 0.0f;
    } else {
#pragma unroll
      for (int i = 0; i < RP; ++i)
#pragma unroll
        for (int j = 0; j < NC; ++j) {
          const int row = r0 + i;
          m[i][j] = (live && row < N && j < N) ? sm[row * N + j] : 0.0f;
        }
      if constexpr (INPL) __syncwarp();         // the matrix's threads have read the slot
#pragma unroll
      for (int i = 0; i < RP; ++i)
        if (r0 + i < N) {
#pragma unroll
          for (int q = 0; q < NCR; ++q)
            *reinterpret_cast<float4 *>(b0 + f32p_off<NCS>(r0 + i, q)) =
                make_float4(m[i][4 * q], m[i][4 * q + 1], m[i][4 * q + 2], m[i][4 * q + 3]);
        }
      __syncwarp();
    }
#pragma unroll 1
    for (int r = 0; r < repeat; ++r) {
      const char *cur = (r & 1) ? b1 : b0;
      char *nxt = (r & 1) ? b0 : b1;
#pragma unroll
      for (int h = 0; h < HALVES; ++h) {
        constexpr int QMAX = QH;
        const int qlo = h * QH;
        const int qn = (NCR - qlo) < QH ? (NCR - qlo) : QH;
        float2 p[RP][2 * QMAX];
#pragma unroll
        for (int i = 0; i < RP; ++i)
#pragma unroll
          for (int jp = 0; jp < 2 * QMAX; ++jp)
            if (jp < 2 * qn) p[i][jp] = make_float2(m[i][4 * qlo + 2 * jp], m[i][4 * qlo + 2 * jp + 1]);
#pragma unroll
        for (int k = 0; k < N; ++k) {
          // keep ptxas from hoisting every row-k load of the group at once
          // (register pressure next to the 4 resident rows)
          if (k % F32P_KSTEP == 0) asm volatile("" ::: "memory");
          float b[4 * QMAX];
#pragma unroll
          for (int q = 0; q < QMAX; ++q)
            if (q < qn) {
              const float4 v = *reinterpret_cast<const float4 *>(cur + f32p_off<NCS>(k, qlo + q));
              b[4 * q] = v.x; b[4 * q + 1] = v.y; b[4 * q + 2] = v.z; b[4 * q + 3] = v.w;
            }
#pragma unroll
          for (int i = 0; i < RP; ++i)
#pragma unroll
            for (int jp = 0; jp < 2 * QMAX; ++jp)
              if (jp < 2 * qn)
                p[i][jp] = __ffma2_rn(make_float2(m[i][k], m[i][k]),
                                      make_float2(b[2 * jp], b[2 * jp + 1]), p[i][jp]);
        }
        // M' = A + c * P (padding stays zero) -> next buffer
#pragma unroll
        for (int i = 0; i < RP; ++i) {
          const int row = r0 + i;
#pragma unroll
          for (int q = 0; q < QMAX; ++q)
            if (q < qn) {
              // the diagonal element of row r0+i sits in chunk tg, lane e == i
              const bool dchunk = (qlo + q) == tg;
              float v[4];
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const int col = 4 * (qlo + q) + e;
                const float pv = (e & 1) ? p[i][2 * q + e / 2].y : p[i][2 * q + e / 2].x;
                const bool diag = (RP == 4) ? (e == i && dchunk) : (col == row);
                const float a = (A == Addend::Ones || diag) ? 1.0f : 0.0f;
                v[e] = ((G * RP == N || row < N) && col < N) ? fmaT(c, pv, a) : 0.0f;
              }
              if (row < N)
                *reinterpret_cast<float4 *>(nxt + f32p_off<NCS>(row, qlo + q)) =
                    make_float4(v[0], v[1], v[2], v[3]);
              if constexpr (HALVES == 1) {
#pragma unroll
                for (int e = 0; e < 4; ++e) m[i][4 * (qlo + q) + e] = v[e];
              }
            }
        }
      }
      if constexpr (HALVES > 1) {   // own rows back from the next buffer (written by this thread)
#pragma unroll
        for (int i = 0; i < RP; ++i)
          if (r0 + i < N) {
#pragma unroll
            for (int q = 0; q < NCR; ++q) {
              const float4 v = *reinterpret_cast<const float4 *>(nxt + f32p_off<NCS>(r0 + i, q));
              m[i][4 * q] = v.x; m[i][4 * q + 1] = v.y; m[i][4 * q + 2] = v.z; m[i][4 * q + 3] = v.w;
            }
          }
      }
      __syncwarp();
    }
    if constexpr (VCP) {   // the final M is the buffer the last update wrote: back to the packed slots
      const int fb = (repeat & 1) ? MBUF : 0;
#pragma unroll 4
      for (int e = lane; e < MPW * CPM; e += 32) {
        const int ml = e / CPM, cc = e - ml * CPM, row = cc / NCR, q = cc - row * NCR, ms = warp * MPW + ml;
        if (ms < cnt)
          *reinterpret_cast<float4 *>(stage + ms * Stg::SBM + cc * 16) =
              *reinterpret_cast<const float4 *>(smem + Stg::BYTES + ms * PSTR + fb + f32p_off<NCS>(row, q));
      }
    } else if (live) {
#pragma unroll
      for (int i = 0; i < RP; ++i)
#pragma unroll
        for (int j = 0; j < NC; ++j) {
          const int row = r0 + i;
          if (row < N && j < N) sm[row * N + j] = m[i][j];
        }
    }
    sg.release();
  }
  sg.finish();
}

// ======================================================================
// F32T (r02; 17 <= n <= 64): FP32 register-tiled outer products with FFMA2,
// sized for occupancy (jm_plan.h F32T).  The RG x CG threads of a matrix each
// own an RA x CB block of P = M + M*M (rows i*RG + tr, 16-B column chunks
// f32t_chunk(h, tc)); accumulators start at M, so P is the only state.  Per
// update: publish M (row stride LDM) over the matrix's region, sync, then for
// every k: P[i][:] += M[i][k] * M[k][:] with the A operand from a per-row
// LDS.128 of M[i][kb..kb+3] (reloaded right after its last use at kk = 3) and
// the B operand, row k, loaded one k ahead; k steps in [N, rup(N, 4)) are not
// computed (their A values are zero padding).  Epilogue M' = A + c*P in FFMA2
// pairs.  Matrices of <= 32 threads share a warp (__syncwarp); 64-thread
// matrices sync their two warps with a named barrier.
// ======================================================================
__device__ __forceinline__ void bar_named(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
// named barrier that also ORs a predicate over its threads
__device__ __forceinline__ bool bar_red_or(int id, int nthreads, bool v) {
  unsigned r;
  asm volatile("{\n\t.reg .pred q, p;\n\tsetp.ne.u32 q, %1, 0;\n\tbarrier.red.or.pred p, %2, %3, q;\n\t"
               "selp.u32 %0, 1, 0, p;\n\t}"
               : "=r"(r) : "r"((unsigned)v), "r"(id), "r"(nthreads) : "memory");
  return r != 0;
}
// 32-bit shared-window addresses throughout: NVRTC otherwise keeps the
// work-area pointers as 64-bit generic addresses (r02: 166 vs 132 registers
// for the same n = 32 kernel built by nvcc, which infers the shared space)
__device__ __forceinline__ float4 lds128(unsigned a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts128(unsigned a, float x, float y, float z, float w) {
  asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(a), "f"(x), "f"(y), "f"(z), "f"(w) : "memory");
}

// v[h] <- v[(h - d) mod NH] (RIGHT: undo a load order that started at chunk
// d) or v[h] <- v[(h + d) mod NH] (left), d < NH a runtime amount: one
// compile-time rotation by 2^b per bit of d, selected at run time
template <int NH, bool RIGHT>
__device__ __forceinline__ void rot_chunks(float4 (&v)[NH], int d) {
#pragma unroll
  for (int b = 1; b < NH; b <<= 1) {
    const bool on = (d & b) != 0;
    float4 w[NH];
#pragma unroll
    for (int h = 0; h < NH; ++h) w[h] = RIGHT ? v[(h - b % NH + NH) % NH] : v[(h + b) % NH];
#pragma unroll
    for (int h = 0; h < NH; ++h) {
      v[h].x = on ? w[h].x : v[h].x;
      v[h].y = on ? w[h].y : v[h].y;
      v[h].z = on ? w[h].z : v[h].z;
      v[h].w = on ? w[h].w : v[h].w;
    }
  }
}

template <int N, Addend A, bool STRM>
__device__ __forceinline__ void run_f32t(const float *__restrict__ in, float *__restrict__ out,
                                         long long batch, int repeat) {
  constexpr int DT = STRM ? 2 : 0;   // the streaming kernel may have its own shape (jm_plan.h F32TS_TABLE)
  constexpr F32T TL = f32t_tile(N, DT);
  constexpr int RA = TL.ra, CB = TL.cb, RG = TL.rg, CG = TL.cg, NH = CB / 4, LDM = TL.ldm;
  constexpr int TPMAT = RG * CG, WPM = f32t_wpm(N, DT), MPW = f32t_mpw(N, DT), WPC = f32t_wpc(N, DT);
  constexpr int MPC = f32t_mpc(N, DT), NR = f32t_nr(N, DT), NC = CG * CB, SROWS = f32t_srows(N, DT);
  constexpr int REG = f32t_region(N, DT), ES = 4, MB = N * N * 4, NT = 32 * WPC;
  constexpr bool AL = ((MPC * MB) % 16) == 0;
  constexpr bool PAD = (NR != N) || (NC != N);
  static_assert(CB % 4 == 0 && NC >= f32t_kp(N, DT), "tile shape");
  static_assert(TL.pack || WPC % WPM == 0, "whole matrices per CTA");
  extern __shared__ __align__(16) char smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // matrix slot in the chunk (mi) and thread index within the matrix (t)
  // (qmix: the two matrices of a warp alternate by quarter-warp, so the two
  // quarters of a half-warp always read different matrices: disjoint
  // addresses, one wavefront per half for both the A and the B loads)
  // (PACK, jm_plan.h F32T.pack: matrices laid end to end over the CTA's
  // threads, straddling warps; CTA barriers)
  constexpr bool PACK = TL.pack;
  const int m = WPM == 1 ? (TL.qmix ? (lane >> 3) & 1 : lane / TPMAT) : 0;
  const int t = PACK ? tid % TPMAT : WPM == 1 ? (TL.qmix ? ((lane >> 4) << 3) + (lane & 7) : lane - m * TPMAT) : (warp % WPM) * 32 + lane;
  const int mi = PACK ? tid / TPMAT : WPM == 1 ? warp * MPW + m : warp / WPM;
  // lanes past the last whole matrix of a warp, or past RG*CG in a multi-warp
  // matrix, idle (but take part in the syncs)
  const bool lane_ok = PACK ? mi < MPC : WPM > 1 ? t < TPMAT : (m < MPW && t < TPMAT);
  const int tr = TL.trfast ? t % RG : t / CG, tc = TL.trfast ? t / RG : t % CG;
  const float c = float(0.00005);
  auto sync = [&]() {
    if constexpr (PACK) __syncthreads();
    else if constexpr (WPM == 1) __syncwarp();
    else if constexpr (WPM == WPC) __syncthreads();
    else bar_named(1 + mi, 32 * WPM);
  };
  auto row_of = [&](int i) { return i * RG + tr; };
  auto chunk_of = [&](int h) { return TL.colblk ? tc * NH + h : h * CG + tc; };
  // PVEC (r02): the one-time read of the staged (packed, row stride N)
  // matrix into the accumulators and the write-back go as 16-B accesses when
  // rows are whole chunks; thread tr takes its NH chunks of a row starting at
  // chunk tr % NH, so the threads of a quarter-warp that share a column
  // (rows 2^k x 16 B apart: one bank slot) touch different chunks at a time.
  // The element accesses were 8-way conflicted at n = 32 (53 % of the R = 1
  // kernel's wavefronts, profiles/r02_ncu_kinds.md).
  constexpr bool PVEC = f32t_pvec(N, STRM);
  const int prot = NH > 1 ? tr % NH : 0;
  // STRM (the low-repeat variant): even n run behind the bulk-copy ring with
  // each slot widened to the work region (f32t_ring); odd n keep the
  // double-buffered cp.async stage (the next chunk streams in while this one
  // is updated)
  // (n % 4 == 0: the ring copies each row straight into the work layout (row
  // pitch LDM), so the matrix is read into the accumulators and written back
  // with conflict-free 16-B accesses in the publish pattern instead of
  // element accesses of the packed layout, whose rows 2^k x 16 B apart put a
  // quarter-warp on one bank: 53 % of the n = 32, R = 1 kernel's wavefronts
  // conflicted, profiles/r02_ncu_kinds.md)
  constexpr bool RROWS = STRM && f32t_ring(N) && JM_F32T_RING_ROWS && (N % 4) == 0;
  // RSEP (f32t_ring_sep): the ring slots hold the packed matrices (one bulk
  // copy per matrix for even n, one per chunk for odd n) and each matrix of
  // the round has its own work region beside the ring.  The threads of a
  // matrix group (a warp, or the warps of one matrix) copy the packed slots
  // into the work layout with consecutive 16-B (n % 4 == 0) or 4-B accesses
  // -- bank-conflict free on both sides -- and the matrix is read into the
  // accumulators, and written back, in the publish pattern; the group copies
  // the result back to the slots for the bulk store.  Per matrix in flight:
  // two packed slots + one work region (the in-place ring: two work regions).
  constexpr bool RSEP = STRM && !f32t_ring(N) && f32t_ring_sep(N);
  // PSH (r02, jm_plan.h f32t_pshift): odd n behind the prefetching stage stage
  // each matrix at byte (global offset & 15) of its region so it moves by
  // 16-B copies in and out (Stager SHIFT) instead of one 4-B copy per element;
  // the packed matrix is read from, and the result written back to, that offset
  constexpr bool PSH = STRM && !f32t_ring(N) && !RSEP && f32t_pshift(N);
  constexpr int GS = 32 * WPM, GM = WPM == 1 ? MPW : 1;   // group threads, group matrices
  const int gt = WPM == 1 ? lane : (warp % WPM) * 32 + lane;
  const int gm0 = WPM == 1 ? warp * MPW : warp / WPM;   // the group's first matrix slot
  typedef typename Pick<STRM && (f32t_ring(N) || RSEP),
                        Ring<N, ES, NT, MPC, ring_kr(N, ES, MPC), JM_RING_S, RSEP ? 0 : REG, RROWS ? LDM * 4 : 0>,
                        Stager<N, ES, REG, NT, MPC, AL, STRM, PSH>>::type Stg;
  static_assert(RSEP || Stg::SBM >= REG, "a slot holds the work region");
  static_assert(!(RSEP && PACK), "the packed-slot copy assumes warp-aligned matrix groups");
  Stg sg(in, out, batch, smem);
  for (sg.start(); sg.valid(); sg.next()) {
    sg.acquire();
    const bool live = lane_ok && mi < sg.cnt();
    int shb = 0;                       // (PSH) the staged matrix's byte offset in its region
    if constexpr (PSH) shb = sg.shift(lane_ok ? mi : 0);
    float *sm = reinterpret_cast<float *>(sg.buf() + (lane_ok ? mi : 0) * Stg::SBM + shb);   // the staged matrix
    float *wk = RSEP ? reinterpret_cast<float *>(smem + Stg::BYTES + (lane_ok ? mi : 0) * REG)
                     : reinterpret_cast<float *>(sg.buf() + (lane_ok ? mi : 0) * Stg::SBM);   // work region
    const unsigned sbase = smem_u32(wk);
    float2 p[RA][CB / 2];
    if constexpr (RSEP) {
      const int cnt = sg.cnt();
      if constexpr (N % 4 == 0) {
        constexpr int CPR = N / 4, CPM = N * CPR;
#pragma unroll 4
        for (int e = gt; e < GM * CPM; e += GS) {
          const int ml = e / CPM, cc = e - ml * CPM, row = cc / CPR, q = cc - row * CPR, ms = gm0 + ml;
          if (ms < cnt)
            *reinterpret_cast<float4 *>(smem + Stg::BYTES + ms * REG + (row * LDM + 4 * q) * 4) =
                *reinterpret_cast<const float4 *>(sg.buf() + ms * Stg::SBM + cc * 16);
        }
      } else {
        constexpr int EPM = N * N;
#pragma unroll 4
        for (int e = gt; e < GM * EPM; e += GS) {
          const int ml = e / EPM, cc = e - ml * EPM, row = cc / N, col = cc - row * N, ms = gm0 + ml;
          if (ms < cnt)
            reinterpret_cast<float *>(smem + Stg::BYTES + ms * REG)[row * LDM + col] =
                reinterpret_cast<const float *>(sg.buf() + ms * Stg::SBM)[cc];
        }
      }
      sync();
#pragma unroll
      for (int i = 0; i < RA; ++i)
#pragma unroll
        for (int h = 0; h < NH; ++h) {
          const int row = row_of(i), c0 = chunk_of(h) * 4;
          float4 v = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
          if (live && row < N && c0 < N) {
            v = lds128(sbase + (row * LDM + c0) * 4);
            if constexpr (N % 4 != 0) {   // the padding columns of the work region hold stale values
              if (c0 + 1 >= N) v.y = 0.0f;
              if (c0 + 2 >= N) v.z = 0.0f;
              if (c0 + 3 >= N) v.w = 0.0f;
            }
          }
          p[i][2 * h] = make_float2(v.x, v.y);
          p[i][2 * h + 1] = make_float2(v.z, v.w);
        }
    } else if constexpr (RROWS) {   // own block of the staged matrix (row-pitched: already the work layout)
#pragma unroll
      for (int i = 0; i < RA; ++i)
#pragma unroll
        for (int h = 0; h < NH; ++h) {
          const int row = row_of(i), c0 = chunk_of(h) * 4;
          float4 v = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
          if (live && row < N && c0 < N) v = lds128(sbase + (row * LDM + c0) * 4);
          p[i][2 * h] = make_float2(v.x, v.y);
          p[i][2 * h + 1] = make_float2(v.z, v.w);
        }
    } else if constexpr (PVEC) {   // packed, rows of whole 16-B chunks: rotated LDS.128 (PVEC above)
      const unsigned pbase = smem_u32(sm);
#pragma unroll
      for (int i = 0; i < RA; ++i) {
        const int row = row_of(i);
        float4 v[NH];
#pragma unroll
        for (int st = 0; st < NH; ++st) {
          const int c0 = chunk_of((st + prot) % NH) * 4;
          v[st] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
          if (live && row < N && c0 < N) v[st] = lds128(pbase + (row * N + c0) * 4);
        }
        rot_chunks<NH, true>(v, prot);   // v[h] = chunk h
#pragma unroll
        for (int h = 0; h < NH; ++h) {
          p[i][2 * h] = make_float2(v[h].x, v[h].y);
          p[i][2 * h + 1] = make_float2(v[h].z, v[h].w);
        }
      }
    } else {   // own block of the staged matrix (packed, row stride N)
#pragma unroll
      for (int i = 0; i < RA; ++i)
#pragma unroll
        for (int h = 0; h < NH; ++h)
#pragma unroll
          for (int e = 0; e < 4; e += 2) {
            const int row = row_of(i), c0 = chunk_of(h) * 4 + e;
            p[i][2 * h + e / 2].x = (live && row < N && c0 < N) ? sm[row * N + c0] : 0.0f;
            p[i][2 * h + e / 2].y = (live && row < N && c0 + 1 < N) ? sm[row * N + c0 + 1] : 0.0f;
          }
    }
    sync();                            // staged matrix read: the region becomes the work area
    if constexpr (SROWS > NR) {        // rows read as k padding (k in [NR, KP)) are zero
      if (live)
        for (int e = t; e < (SROWS - NR) * LDM; e += TPMAT) wk[NR * LDM + e] = 0.0f;
    }
    for (int r = 0; r < repeat; ++r) {
      if (live) {                      // publish M
#pragma unroll
        for (int i = 0; i < RA; ++i)
#pragma unroll
          for (int h = 0; h < NH; ++h)
            sts128(sbase + (row_of(i) * LDM + chunk_of(h) * 4) * 4, p[i][2 * h].x, p[i][2 * h].y,
                   p[i][2 * h + 1].x, p[i][2 * h + 1].y);
      }
      sync();
      if (live) {
        const unsigned bcol = sbase + chunk_of(0) * 16;   // B: row k at bcol + k*LDM*4
        float4 bq[NH], bn[NH];
#pragma unroll
        for (int h = 0; h < NH; ++h) bq[h] = lds128(bcol + (chunk_of(h) - chunk_of(0)) * 16);
        // A: row i*RG + tr at arow + i*RG*LDM*4, four k values per LDS.128,
        // each row's block reloaded right after its last use
        const unsigned arow = sbase + tr * LDM * 4;
        float4 av[RA];
#pragma unroll
        for (int i = 0; i < RA; ++i) av[i] = lds128(arow + i * RG * LDM * 4);
        // full blocks of four k steps (rolled above n ~ 48: the fully
        // unrolled update overflows the instruction cache), then N % 4
        constexpr int KF = N / 4, KT = N % 4;
        auto kstep = [&](int k, int kk, bool more, bool reload_a) {
          if (more) {
#pragma unroll
            for (int h = 0; h < NH; ++h)
              bn[h] = lds128(bcol + (k + 1) * LDM * 4 + (chunk_of(h) - chunk_of(0)) * 16);
          }
#pragma unroll
          for (int i = 0; i < RA; ++i) {
            const float a = kk == 0 ? av[i].x : kk == 1 ? av[i].y : kk == 2 ? av[i].z : av[i].w;
#pragma unroll
            for (int h = 0; h < NH; ++h) {
              p[i][2 * h] = __ffma2_rn(make_float2(a, a), make_float2(bq[h].x, bq[h].y), p[i][2 * h]);
              p[i][2 * h + 1] = __ffma2_rn(make_float2(a, a), make_float2(bq[h].z, bq[h].w), p[i][2 * h + 1]);
            }
            if (reload_a) av[i] = lds128(arow + i * RG * LDM * 4 + (k + 1) * 4);
          }
#pragma unroll
          for (int h = 0; h < NH; ++h) bq[h] = bn[h];
        };
        constexpr int KU = f32t_kunroll(N, DT);
#pragma unroll KU
        for (int kb = 0; kb < KF; ++kb) {
          const bool last = kb == KF - 1;
          kstep(4 * kb + 0, 0, true, false);
          kstep(4 * kb + 1, 1, true, false);
          kstep(4 * kb + 2, 2, true, false);
          kstep(4 * kb + 3, 3, !last || KT > 0, !last || KT > 0);
        }
#pragma unroll
        for (int kk = 0; kk < KT; ++kk) kstep(4 * KF + kk, kk, kk + 1 < KT, false);
      }
      sync();                          // every read of this update's M done before the next publish
      if (live) {
        const float2 c2 = make_float2(c, c);
#pragma unroll
        for (int i = 0; i < RA; ++i)
#pragma unroll
          for (int j = 0; j < CB / 2; ++j) {
            const int row = row_of(i), c0 = chunk_of(j / 2) * 4 + 2 * (j & 1);
            float2 a2 = make_float2(1.0f, 1.0f);
            if constexpr (A == Addend::Identity) a2 = make_float2(row == c0 ? 1.0f : 0.0f, row == c0 + 1 ? 1.0f : 0.0f);
            float2 q = __ffma2_rn(c2, p[i][j], a2);
            if constexpr (PAD) {         // padding stays exactly zero
              if (row >= N || c0 >= N) q.x = 0.0f;
              if (row >= N || c0 + 1 >= N) q.y = 0.0f;
            }
            p[i][j] = q;
          }
      }
    }
    if constexpr (RSEP) {              // work layout (publish pattern), then the group copies it to the slots
      if (live) {
#pragma unroll
        for (int i = 0; i < RA; ++i)
#pragma unroll
          for (int h = 0; h < NH; ++h) {
            const int row = row_of(i), c0 = chunk_of(h) * 4;
            if (row < N && c0 < N)
              sts128(sbase + (row * LDM + c0) * 4, p[i][2 * h].x, p[i][2 * h].y, p[i][2 * h + 1].x,
                     p[i][2 * h + 1].y);
          }
      }
      sync();
      const int cnt = sg.cnt();
      if constexpr (N % 4 == 0) {
        constexpr int CPR = N / 4, CPM = N * CPR;
#pragma unroll 4
        for (int e = gt; e < GM * CPM; e += GS) {
          const int ml = e / CPM, cc = e - ml * CPM, row = cc / CPR, q = cc - row * CPR, ms = gm0 + ml;
          if (ms < cnt)
            *reinterpret_cast<float4 *>(sg.buf() + ms * Stg::SBM + cc * 16) =
                *reinterpret_cast<const float4 *>(smem + Stg::BYTES + ms * REG + (row * LDM + 4 * q) * 4);
        }
      } else {
        constexpr int EPM = N * N;
#pragma unroll 4
        for (int e = gt; e < GM * EPM; e += GS) {
          const int ml = e / EPM, cc = e - ml * EPM, row = cc / N, col = cc - row * N, ms = gm0 + ml;
          if (ms < cnt)
            reinterpret_cast<float *>(sg.buf() + ms * Stg::SBM)[cc] =
                reinterpret_cast<const float *>(smem + Stg::BYTES + ms * REG)[row * LDM + col];
        }
      }
    } else if constexpr (RROWS) {      // rows leave from the work layout (the k loop's reads are done)
      if (live) {
#pragma unroll
        for (int i = 0; i < RA; ++i)
#pragma unroll
          for (int h = 0; h < NH; ++h) {
            const int row = row_of(i), c0 = chunk_of(h) * 4;
            if (row < N && c0 < N)
              sts128(sbase + (row * LDM + c0) * 4, p[i][2 * h].x, p[i][2 * h].y, p[i][2 * h + 1].x,
                     p[i][2 * h + 1].y);
          }
      }
    } else if (PVEC && live) {         // back to the packed layout: rotated STS.128
      const unsigned pbase = smem_u32(sm);
#pragma unroll
      for (int i = 0; i < RA; ++i) {
        const int row = row_of(i);
        float4 v[NH];
#pragma unroll
        for (int h = 0; h < NH; ++h) v[h] = make_float4(p[i][2 * h].x, p[i][2 * h].y, p[i][2 * h + 1].x, p[i][2 * h + 1].y);
        rot_chunks<NH, false>(v, prot);  // v[st] = chunk (st + prot) % NH
#pragma unroll
        for (int st = 0; st < NH; ++st) {
          const int c0 = chunk_of((st + prot) % NH) * 4;
          if (row < N && c0 < N) sts128(pbase + (row * N + c0) * 4, v[st].x, v[st].y, v[st].z, v[st].w);
        }
      }
    } else if (live) {                 // back to the packed layout for the store
#pragma unroll
      for (int i = 0; i < RA; ++i)
#pragma unroll
        for (int h = 0; h < NH; ++h)
#pragma unroll
          for (int e = 0; e < 4; e += 2) {
            const int row = row_of(i), c0 = chunk_of(h) * 4 + e;
            if (row < N && c0 < N) sm[row * N + c0] = p[i][2 * h + e / 2].x;
            if (row < N && c0 + 1 < N) sm[row * N + c0 + 1] = p[i][2 * h + e / 2].y;
          }
    }
    sg.release();
  }
  sg.finish();
}

// ======================================================================
// F64T (r02): FP64 register tiles with DFMA, for the sizes where DMMA's
// 8 x 8 x 4 granularity wastes most of the FP64 pipe (jm_plan.h F64T_TABLE).
// The same scheme as run_f32t with a 16-B chunk holding two doubles: thread
// (tr, tc) owns an RA x CB block of P; per k, A = M[i][k] from a per-row
// LDS.128 of M[i][2kb..2kb+1] (reloaded after its last use at kk = 1) and B =
// row k one k ahead; DFMA and DMMA share the FP64 pipe (64 FMA/clk/SM), so
// padding only to multiples of the register tile (not of 8) is the gain.
// ======================================================================
__device__ __forceinline__ double2 lds128d(unsigned a) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts128d(unsigned a, double x, double y) {
  asm volatile("st.shared.v2.f64 [%0], {%1,%2};" ::"r"(a), "d"(x), "d"(y) : "memory");
}

template <int N, Addend A, bool STRM>
__device__ __forceinline__ void run_f64t(const double *__restrict__ in, double *__restrict__ out,
                                         long long batch, int repeat) {
  constexpr F32T TL = f32t_tile(N, 1);
  constexpr int RA = TL.ra, CB = TL.cb, RG = TL.rg, CG = TL.cg, NH = CB / 2, LDM = TL.ldm;
  constexpr int TPMAT = RG * CG, WPM = f32t_wpm(N, 1), MPW = f32t_mpw(N, 1), WPC = f32t_wpc(N, 1);
  constexpr int MPC = f32t_mpc(N, 1), NR = f32t_nr(N, 1), NC = CG * CB, SROWS = f32t_srows(N, 1);
  constexpr int REG = f32t_region(N, 1), ES = 8, MB = N * N * 8, NT = 32 * WPC;
  constexpr bool AL = ((MPC * MB) % 16) == 0;
  constexpr bool PAD = (NR != N) || (NC != N);
  static_assert(CB % 2 == 0 && NC >= f32t_kp(N, 1), "tile shape");
  static_assert(TL.pack || WPC % WPM == 0, "whole matrices per CTA");
  extern __shared__ __align__(16) char smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr bool PACK = TL.pack;   // (lane-packed CTA, jm_plan.h F32T.pack)
  const int m = WPM == 1 ? (TL.qmix ? (lane >> 3) & 1 : lane / TPMAT) : 0;
  const int t = PACK ? tid % TPMAT : WPM == 1 ? (TL.qmix ? ((lane >> 4) << 3) + (lane & 7) : lane - m * TPMAT) : (warp % WPM) * 32 + lane;
  const int mi = PACK ? tid / TPMAT : WPM == 1 ? warp * MPW + m : warp / WPM;
  const bool lane_ok = PACK ? mi < MPC : WPM > 1 ? t < TPMAT : (m < MPW && t < TPMAT);
  const int tr = TL.trfast ? t % RG : t / CG, tc = TL.trfast ? t / RG : t % CG;
  const double c = 0.00005;
  auto sync = [&]() {
    if constexpr (PACK) __syncthreads();
    else if constexpr (WPM == 1) __syncwarp();
    else if constexpr (WPM == WPC) __syncthreads();
    else bar_named(1 + mi, 32 * WPM);
  };
  auto row_of = [&](int i) { return i * RG + tr; };
  auto chunk_of = [&](int h) { return TL.colblk ? tc * NH + h : h * CG + tc; };
  Stager<N, ES, REG, NT, MPC, AL, STRM> sg(in, out, batch, smem);
  for (sg.start(); sg.valid(); sg.next()) {
    sg.acquire();
    const bool live = lane_ok && mi < sg.cnt();
    double *sm = reinterpret_cast<double *>(sg.buf() + (lane_ok ? mi : 0) * REG);
    const unsigned sbase = smem_u32(sm);
    double p[RA][CB];
#pragma unroll
    for (int i = 0; i < RA; ++i)
#pragma unroll
      for (int j = 0; j < CB; ++j) {
        const int row = row_of(i), col = chunk_of(j / 2) * 2 + (j & 1);
        p[i][j] = (live && row < N && col < N) ? sm[row * N + col] : 0.0;
      }
    sync();
    if constexpr (SROWS > NR) {
      if (live)
        for (int e = t; e < (SROWS - NR) * LDM; e += TPMAT) sm[NR * LDM + e] = 0.0;
    }
    for (int r = 0; r < repeat; ++r) {
      if (live) {
#pragma unroll
        for (int i = 0; i < RA; ++i)
#pragma unroll
          for (int h = 0; h < NH; ++h) sts128d(sbase + (row_of(i) * LDM + chunk_of(h) * 2) * 8, p[i][2 * h], p[i][2 * h + 1]);
      }
      sync();
      if (live) {
        const unsigned bcol = sbase + chunk_of(0) * 16;
        double2 bq[NH], bn[NH];
#pragma unroll
        for (int h = 0; h < NH; ++h) bq[h] = lds128d(bcol + (chunk_of(h) - chunk_of(0)) * 16);
        const unsigned arow = sbase + tr * LDM * 8;
        double2 av[RA];
#pragma unroll
        for (int i = 0; i < RA; ++i) av[i] = lds128d(arow + i * RG * LDM * 8);
        constexpr int KF = N / 2, KT = N % 2;
        auto kstep = [&](int k, int kk, bool more, bool reload_a) {
          if (more) {
#pragma unroll
            for (int h = 0; h < NH; ++h)
              bn[h] = lds128d(bcol + (k + 1) * LDM * 8 + (chunk_of(h) - chunk_of(0)) * 16);
          }
#pragma unroll
          for (int i = 0; i < RA; ++i) {
            const double a = kk == 0 ? av[i].x : av[i].y;
#pragma unroll
            for (int h = 0; h < NH; ++h) {
              p[i][2 * h] = fmaT(a, bq[h].x, p[i][2 * h]);
              p[i][2 * h + 1] = fmaT(a, bq[h].y, p[i][2 * h + 1]);
            }
            if (reload_a) av[i] = lds128d(arow + i * RG * LDM * 8 + (k + 1) * 8);
          }
#pragma unroll
          for (int h = 0; h < NH; ++h) bq[h] = bn[h];
        };
        constexpr int KU = f32t_kunroll(N, 1);
#pragma unroll KU
        for (int kb = 0; kb < KF; ++kb) {
          const bool last = kb == KF - 1;
          kstep(2 * kb + 0, 0, true, false);
          kstep(2 * kb + 1, 1, !last || KT > 0, !last || KT > 0);
        }
        if constexpr (KT > 0) kstep(2 * KF, 0, false, false);
      }
      sync();
      if (live) {
#pragma unroll
        for (int i = 0; i < RA; ++i)
#pragma unroll
          for (int j = 0; j < CB; ++j) {
            const int row = row_of(i), col = chunk_of(j / 2) * 2 + (j & 1);
            const double a = (A == Addend::Ones || row == col) ? 1.0 : 0.0;
            double v = fmaT(c, p[i][j], a);
            if constexpr (PAD) v = (row < N && col < N) ? v : 0.0;
            p[i][j] = v;
          }
      }
    }
    if (live) {
#pragma unroll
      for (int i = 0; i < RA; ++i)
#pragma unroll
        for (int j = 0; j < CB; ++j) {
          const int row = row_of(i), col = chunk_of(j / 2) * 2 + (j & 1);
          if (row < N && col < N) sm[row * N + col] = p[i][j];
        }
    }
    sg.release();
  }
  sg.finish();
}

// ======================================================================
// run_f32tc — FP32 on the tensor cores (jm_plan.h f32tc_use): a warp per
// matrix, n = 16*MT.  Lane (g, t) = (lane / 4, lane % 4) holds, for m-tile I
// and n-tile J, the m16n8 accumulator fragment {(16I+g, 8J+2t), (.., 8J+2t+1),
// (16I+g+8, 8J+2t), (.., 8J+2t+1)} of M (then of P = M + M.M).  Under the k
// permutation (t, t+4) -> (2t, 2t+1) within a k-step, n-tile KS's fragment is
// the m16n8k8 A fragment {a0, a1, a2, a3} = {c0, c2, c1, c3} of k-step KS, so
// only the B operand B[k][j] = M[8KS + 2t (+1)][8J + g] is read from the
// warp's published copy of M.  Each operand x is split x = hi + lo (hi, lo
// TF32; tf32_split) and lo.hi + hi.lo + hi.hi accumulate in FP32 (the 3xTF32
// scheme; lo.lo ~ 2^-21 relative is dropped).
// ======================================================================
// The split without cvt.rna.tf32 (an FSETP / VIADD / LOP3 / SEL sequence per
// value in SASS, which made the ALU pipe the bound): hi = x with the 13 low
// mantissa bits cleared (exact: lo = x - hi is exact in FP32), lo rounded to
// TF32 by adding half an ulp and clearing the same bits (lo is finite and
// far from overflow), or (JM_F32TC_LORND=0, the default) passed as is, the
// mma reading it truncated: measured max relative error vs the oracle 1.6e-6
// (rounded: 1.3e-6) against the 1e-5 FP32 bound, 0.931 vs 0.914 of the FP32
// pipe at n = 32 (profiles/r02_f32tc.md).
#ifndef JM_F32TC_LORND
#define JM_F32TC_LORND 0
#endif
#ifndef JM_F32TC_SAFE
#define JM_F32TC_SAFE 1   // 0: no exact-path check (timing experiment only: wrong near overflow / infinities)
#endif
// (hi is formed as x - (x - mask(x)), exactly mask(x): ptxas knows the mma
// ignores the low bits, so a plain mask operand became the raw accumulator and
// the permuted A quad was rebuilt with four MOVs at every use; the FADD result
// is allocated in quad order once)
__device__ __forceinline__ void tf32_split(float x, unsigned &hi, unsigned &lo) {
  const float d = x - __uint_as_float(__float_as_uint(x) & 0xffffe000u);   // exact
  hi = __float_as_uint(x - d);                                              // exact: the masked x
  const unsigned l = __float_as_uint(d);
  lo = JM_F32TC_LORND ? (l + 0x1000u) & 0xffffe000u : l;
}
__device__ __forceinline__ void mma_tf32(float (&d)[4], const unsigned (&a)[4], unsigned b0, unsigned b1) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
               "{%0,%1,%2,%3};"
               : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
               : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

template <int N, Addend A>
__device__ __forceinline__ void run_f32tc(const float *__restrict__ in, float *__restrict__ out,
                                          long long batch, int repeat) {
  // (n not a multiple of 8: M is held zero-padded to NP = 8*ceil(n/8), the
  // padding re-zeroed by every epilogue, so it never reaches a real entry)
  constexpr int NP = (N + 7) / 8 * 8;
  // MT m-tiles of this warp (MTW of the matrix's N/16; WPM warps per matrix)
  constexpr int MT = f32tc_mtw(N), WPM = f32tc_wpm(N), NT8 = NP / 8, LD = f32tc_ld(N), MPC = f32tc_mpc(N);
  constexpr int NT = 32 * f32tc_wpc(N), SB = stage_stride(N, 4);
  constexpr bool AL = ((MPC * N * N * 4) % 16) == 0;
  extern __shared__ __align__(16) char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int mi = warp / WPM, r0 = 16 * MT * (warp % WPM);   // matrix slot, first row of this warp
  const float c = float(0.00005);
  auto msync = [&]() {
    if constexpr (WPM == 1) __syncwarp();
    else bar_named(1 + mi, 32 * WPM);
  };
  Stager<N, 4, SB, NT, MPC, AL, false> sg(in, out, batch, smem);
  // entries (row, col), (row, col + 1) of the staged (packed, row stride N) matrix; zero outside it
  auto ld2 = [&](const float *sm, int row, int col) {
    if constexpr (N % 8 == 0) {
      return (N % 16 == 0 || row < N) ? *reinterpret_cast<const float2 *>(sm + row * N + col) : make_float2(0.0f, 0.0f);
    } else {
      return make_float2(row < N && col < N ? sm[row * N + col] : 0.0f, row < N && col + 1 < N ? sm[row * N + col + 1] : 0.0f);
    }
  };
  float *w = reinterpret_cast<float *>(smem + Stager<N, 4, SB, NT, MPC, AL, false>::BYTES) + mi * (16 * f32tc_mt(N)) * LD;
  for (sg.start(); sg.valid(); sg.next()) {
    sg.acquire();
    const bool live = mi < sg.cnt();
    float *sm = reinterpret_cast<float *>(sg.buf() + mi * SB);
    float acc[MT][NT8][4];
    if (live) {
#pragma unroll
      for (int I = 0; I < MT; ++I)
#pragma unroll
        for (int J = 0; J < NT8; ++J)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const float2 v = ld2(sm, r0 + 16 * I + g + 8 * h, 8 * J + 2 * t);
            acc[I][J][2 * h] = v.x;
            acc[I][J][2 * h + 1] = v.y;
          }
      // Exact-path flag (matrix-uniform after the vote below): a matrix with
      // an entry |m| > TM = 1 / (2 c n), or a non-finite one, is expanding
      // (c (1 + 2|M|) > 1: every update amplifies earlier rounding errors),
      // and the 3xTF32 products' small biased error then grows past the bound
      // within a few updates (paper-init inputs: 2e-5 one update before they
      // overflow, FFMA 3e-7; tools/tc_diag_paper.py); such an update runs as
      // the plain FP32 FMA chain instead (k ascending, p = M first: the other
      // kinds' order, so IEEE infinities and NaNs also fall where the
      // oracle's do).  Contracting inputs (c rho < 1) never reach TM.
      constexpr float TM = 0.5f / (0.00005f * N);
      bool bad = false;
#pragma unroll
      for (int I = 0; I < (JM_F32TC_SAFE ? MT : 0); ++I)
#pragma unroll
        for (int J = 0; J < NT8; ++J)
#pragma unroll
          for (int q = 0; q < 4; ++q) bad |= !(fabsf(acc[I][J][q]) <= TM);
      for (int r = 0; r < repeat; ++r) {
        // publish M (row-major, row stride LD) for the B operand
#pragma unroll
        for (int I = 0; I < MT; ++I)
#pragma unroll
          for (int J = 0; J < NT8; ++J)
#pragma unroll
            for (int h = 0; h < 2; ++h)
              *reinterpret_cast<float2 *>(w + (r0 + 16 * I + g + 8 * h) * LD + 8 * J + 2 * t) =
                  make_float2(acc[I][J][2 * h], acc[I][J][2 * h + 1]);
        // A fragments (hi, lo) of every k-step, taken before the products overwrite acc
        unsigned ah[MT][NT8][4], al[MT][NT8][4];
#pragma unroll
        for (int I = 0; I < MT; ++I)
#pragma unroll
          for (int KS = 0; KS < NT8; ++KS)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              tf32_split(acc[I][KS][q == 1 ? 2 : q == 2 ? 1 : q], ah[I][KS][q], al[I][KS][q]);
            }
        bool exact;
        if constexpr (WPM == 1) {
          exact = __any_sync(0xffffffffu, bad);
          __syncwarp();
        } else {
          exact = bar_red_or(1 + mi, 32 * WPM, bad);   // (the publish barrier, with the vote)
        }
        if (!exact) {
#pragma unroll
        for (int KS = 0; KS < NT8; ++KS) {
          unsigned bh[NT8][2], bl[NT8][2];
#pragma unroll
          for (int J = 0; J < NT8; ++J)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              tf32_split(w[(8 * KS + 2 * t + h) * LD + 8 * J + g], bh[J][h], bl[J][h]);
            }
          // small terms first; consecutive mma on different accumulators
#pragma unroll
          for (int pr = 0; pr < 3; ++pr)
#pragma unroll
            for (int J = 0; J < NT8; ++J)
#pragma unroll
              for (int I = 0; I < MT; ++I) {
                if (pr == 0) mma_tf32(acc[I][J], al[I][KS], bh[J][0], bh[J][1]);
                else if (pr == 1) mma_tf32(acc[I][J], ah[I][KS], bl[J][0], bl[J][1]);
                else mma_tf32(acc[I][J], ah[I][KS], bh[J][0], bh[J][1]);
              }
        }
        }
        if constexpr (WPM == 1) __syncwarp();   // every read of w done before the next publish
        else msync();
        if (exact) {   // (rare: rolled loops, P through the matrix's idle stage slot)
#pragma unroll 1
          for (int e = lane; e < 16 * MT * N; e += 32) {
            const int row = r0 + e / N, col = e - (e / N) * N;
            if (N % 16 != 0 && row >= N) break;   // (padding rows: rows only grow with e)
            float pv = w[row * LD + col];
#pragma unroll 1
            for (int k = 0; k < N; ++k) pv = fmaT(w[row * LD + k], w[k * LD + col], pv);
            sm[row * N + col] = pv;
          }
          __syncwarp();
#pragma unroll
          for (int I = 0; I < MT; ++I)
#pragma unroll
            for (int J = 0; J < NT8; ++J)
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const float2 v = ld2(sm, r0 + 16 * I + g + 8 * h, 8 * J + 2 * t);
                acc[I][J][2 * h] = v.x;
                acc[I][J][2 * h + 1] = v.y;
              }
          msync();
        }
        bad = false;
#pragma unroll
        for (int I = 0; I < MT; ++I)
#pragma unroll
          for (int J = 0; J < NT8; ++J)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const int row = r0 + 16 * I + g + 8 * (q >> 1), col = 8 * J + 2 * t + (q & 1);
              const float a = (A == Addend::Ones || row == col) ? 1.0f : 0.0f;
              acc[I][J][q] = fmaT(c, acc[I][J][q], a);
              if constexpr (N % 8 != 0) acc[I][J][q] = (row < N && col < N) ? acc[I][J][q] : 0.0f;
              if constexpr (JM_F32TC_SAFE) bad |= !(fabsf(acc[I][J][q]) <= TM);
            }
      }
#pragma unroll
      for (int I = 0; I < MT; ++I)
#pragma unroll
        for (int J = 0; J < NT8; ++J)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int row = r0 + 16 * I + g + 8 * h, col = 8 * J + 2 * t;
            if constexpr (N % 8 == 0) {
              if (N % 16 == 0 || row < N)
                *reinterpret_cast<float2 *>(sm + row * N + col) = make_float2(acc[I][J][2 * h], acc[I][J][2 * h + 1]);
            } else {
              if (row < N && col < N) sm[row * N + col] = acc[I][J][2 * h];
              if (row < N && col + 1 < N) sm[row * N + col + 1] = acc[I][J][2 * h + 1];
            }
          }
    }
    sg.release();
  }
  sg.finish();
}

// ------------------------------------------------------------------ entry
// The NVRTC name expression is "jm::k_update<N, T, jm::Addend::X, jm::Tile::Y>"
// with Y = tile_for(N, dtype); the host launches it with plan_specialized().
template <int N, class T, Addend A, Tile K, bool STRM = false>
__device__ __forceinline__ void update_body(const T *__restrict__ in, T *__restrict__ out,
                                            long long batch, int repeat) {
  static_assert(N >= 1 && N <= 64, "N in [1, 64]");
  static_assert(K == tile_for(N, sizeof(T) == 8 ? 1 : 0), "tile must match the plan");
  static_assert(!STRM || stream_ok(N, sizeof(T) == 8 ? 1 : 0), "no streaming variant of this kind");
  if constexpr (K == Tile::TPM) {
    run_tpm<N, T, A, STRM>(in, out, batch, repeat);
  } else if constexpr (K == Tile::Tpms && sizeof(T) == 4) {
    if constexpr (STRM) run_f32p<N, A, true>(in, out, batch, repeat);      // low repeat: row panels + ring
    else run_tpms<N, T, A>(in, out, batch, repeat);
  } else if constexpr (K == Tile::Tpms) {
    if constexpr (STRM) run_dmma<N, A, 1, true>(in, out, batch, repeat);   // low repeat: the DMMA ring
    else run_tpms<N, T, A>(in, out, batch, repeat);
  } else if constexpr (K == Tile::Reg) {
    if constexpr (STRM) run_dmma<N, A, 1, true>(in, out, batch, repeat);   // low repeat: the DMMA ring
    else run_f64t<N, A, false>(in, out, batch, repeat);
  } else if constexpr (K == Tile::Dmma) {
    run_dmma<N, A, dmma_w(N, STRM), STRM>(in, out, batch, repeat);
  } else if constexpr (!STRM && sizeof(T) == 4 && f32tc_use(N)) {
    run_f32tc<N, A>(in, out, batch, repeat);
  } else if constexpr (f32p_use(N) && !(STRM && f32t_stream_use(N))) {
    run_f32p<N, A, STRM>(in, out, batch, repeat);
  } else {
    run_f32t<N, A, STRM>(in, out, batch, repeat);
  }
}

template <int N, class T, Addend A, Tile K>
__global__ void __launch_bounds__(plan_specialized(N, sizeof(T) == 8 ? 1 : 0).threads)
    k_update(const T *__restrict__ in, T *__restrict__ out, long long batch, int repeat) {
  update_body<N, T, A, K>(in, out, batch, repeat);
}

// Same body, with minBlocksPerSM = 1 stated: for the CTA-per-matrix DMMA kinds
// this lets ptxas keep ~180 registers (r01: n=64 spilled 8 B at 168 without it,
// and n=32 ran 0.83 vs 0.91 of the FP64 pipe).  kernel_name_for() selects it.
template <int N, class T, Addend A, Tile K>
__global__ void __launch_bounds__(plan_specialized(N, sizeof(T) == 8 ? 1 : 0).threads, 1)
    k_update_mb1(const T *__restrict__ in, T *__restrict__ out, long long batch, int repeat) {
  update_body<N, T, A, K>(in, out, batch, repeat);
}

// Same body under a register cap instead of launch bounds (CUDA forbids both
// on one kernel): the F32T tiles (jm_plan.h f32t_maxreg).
template <int N, class T, Addend A, Tile K>
__global__ void __maxnreg__(f32t_maxreg(N, sizeof(T) == 8)) k_update_rc(const T *__restrict__ in, T *__restrict__ out,
                                                        long long batch, int repeat) {
  update_body<N, T, A, K>(in, out, batch, repeat);
}

template <int N, class T, Addend A, Tile K>
__global__ void __maxnreg__(f32t_maxreg(N, sizeof(T) == 8 ? 1 : 2)) k_update_stream_rc(const T *__restrict__ in, T *__restrict__ out,
                                                               long long batch, int repeat) {
  update_body<N, T, A, K, true>(in, out, batch, repeat);
}

// Latency path (jm_plan.h plan_lat): one warp per matrix, lane e = i*N + j
// holds M[i][j]; P[i][j] = M[i][j] + sum_k M[i][k] M[k][j] with the k terms
// shuffled in, k ascending with FMA — the thread-per-matrix kernel's order, so
// the two agree bit for bit.  Grid-stride over matrices; the warp index is
// warp-uniform, so whole warps leave together and every shuffle is full-warp.
template <int N, class T, Addend A>
__global__ void __launch_bounds__(LAT_THREADS) k_update_lat(const T *__restrict__ in, T *__restrict__ out,
                                                            long long batch, int repeat) {
  static_assert(N * N <= 32, "one matrix per warp");
  const int lane = threadIdx.x & 31;
  const int e = lane < N * N ? lane : 0, i = e / N, j = e - (e / N) * N;
  const T c = T(0.00005);
  const long long nw = (long long)gridDim.x * (LAT_THREADS / 32);
  for (long long b = (long long)blockIdx.x * (LAT_THREADS / 32) + (threadIdx.x >> 5); b < batch; b += nw) {
    T m = lane < N * N ? in[b * N * N + e] : T(0);
    for (int r = 0; r < repeat; ++r) {
      T p = m;
#pragma unroll
      for (int k = 0; k < N; ++k) {
        const T a = __shfl_sync(0xffffffffu, m, i * N + k);
        const T bk = __shfl_sync(0xffffffffu, m, k * N + j);
        p = fmaT(a, bk, p);
      }
      m = (A == Addend::Ones || i == j) ? fmaT(c, p, T(1)) : c * p;
    }
    if (lane < N * N) out[b * N * N + e] = m;
  }
}

// The streaming (low-repeat) variant: same kinds behind the bulk-copy ring
// (plan_stream); the host selects it when repeat * (n + 1) is below the
// switch point.  Name expression "jm::k_update_stream[_mb1]<N, T, A, K>".
template <int N, class T, Addend A, Tile K>
__global__ void __launch_bounds__(plan_stream(N, sizeof(T) == 8 ? 1 : 0).threads)
    k_update_stream(const T *__restrict__ in, T *__restrict__ out, long long batch, int repeat) {
  update_body<N, T, A, K, true>(in, out, batch, repeat);
}
template <int N, class T, Addend A, Tile K>
__global__ void __launch_bounds__(plan_stream(N, sizeof(T) == 8 ? 1 : 0).threads, 1)
    k_update_stream_mb1(const T *__restrict__ in, T *__restrict__ out, long long batch, int repeat) {
  update_body<N, T, A, K, true>(in, out, batch, repeat);
}

}  // namespace jm
#endif  // JM_UPDATE_CUH
