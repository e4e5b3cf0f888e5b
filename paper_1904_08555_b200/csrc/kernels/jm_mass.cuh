// jm_mass.cuh — Laghos 2D mass-operator action rMassMultAdd2D<D, Q>
// (§5.3, Listing 12; reading R18 in DESIGN.md):
//
//     S = (B X_e B^T) .* op_e ;   Y_e += B^T S B          (per element e)
//
// with B the Q x D dofToQuad basis.  In Laghos the (D, Q) = (NUM_DOFS_1D,
// NUM_QUAD_1D) pair selects one of ~32 explicit instantiations through a
// dispatch map; here NVRTC instantiates jm::k_mass<D, Q> on first use, exactly
// like k_update.  FP64.  Per element 4DQ(D+Q) + Q^2 flops against
// (3D^2 + Q^2) doubles of traffic: HBM-bound at every (D, Q) <= 8, so the
// kernels are streaming ones.  Small D*Q*(D+Q): one thread per element,
// x / op / y chunks staged through shared memory with coalesced 128-bit copies
// at an odd 16-B stride (conflict-free per-thread reads), B in shared memory
// (broadcast reads), the quadrature-point values S in registers.  Larger
// (jm_plan.h mass_dmma): one warp per element on the FP64 tensor cores
// (mass_dmma_body below).  Appended
// to the NVRTC source.
#ifndef JM_MASS_CUH
#define JM_MASS_CUH

namespace jm {

template <int D, int Q>
__device__ __forceinline__ void mass_body(const double *__restrict__ B, const double *__restrict__ op,
                                          const double *__restrict__ x, double *__restrict__ y,
                                          long long elements) {
  constexpr int NT = MASS_THREADS, MPC = MASS_THREADS;
  constexpr int SBX = stage_stride(D, 8), SBQ = stage_stride(Q, 8);
  constexpr int MBX = D * D * 8, MBQ = Q * Q * 8;
  // r02 (JM_MASS_PF): two stage buffers, the next chunk's x / y / op stream in
  // by cp.async while this chunk is computed (the single-buffered kernel was
  // latency-bound: long-scoreboard stalls, profiles/r02_ncu_mass.md)
  constexpr bool PF = mass_pf(D, Q);
  constexpr int SXB = stage_bytes(MPC, D, 8), STB = 2 * SXB + stage_bytes(MPC, Q, 8);
  extern __shared__ __align__(16) char smem[];
  double *sB = reinterpret_cast<double *>(smem + (PF ? 2 : 1) * STB);
  const int tid = threadIdx.x;
  for (int i = tid; i < Q * D; i += NT) sB[i] = B[i];
  const long long nchunks = (elements + MPC - 1) / MPC;
  auto count = [&](long long c) { return (int)((elements - c * MPC) < MPC ? (elements - c * MPC) : MPC); };
  auto issue = [&](long long c, char *st) {
    const long long e0 = c * MPC;
    stage_in_async<D, 8, SBX, NT, true>(reinterpret_cast<const char *>(x) + e0 * MBX, st, count(c), tid);
    stage_in_async<D, 8, SBX, NT, true>(reinterpret_cast<const char *>(y) + e0 * MBX, st + SXB, count(c), tid);
    stage_in_async<Q, 8, SBQ, NT, true>(reinterpret_cast<const char *>(op) + e0 * MBQ, st + 2 * SXB, count(c), tid);
    cp_async_commit();
  };
  if (PF && blockIdx.x < nchunks) issue(blockIdx.x, smem);
  int it = 0;
  for (long long ch = blockIdx.x; ch < nchunks; ch += gridDim.x, ++it) {
    const long long e0 = ch * MPC;
    const int cnt = count(ch);
    char *sx = smem + (PF ? (it & 1) * STB : 0), *sy = sx + SXB, *so = sx + 2 * SXB;
    if constexpr (PF) {
      cp_async_wait_all();
      __syncthreads();   // chunk ch visible; every thread is done with the other buffer
      if (ch + gridDim.x < nchunks) issue(ch + gridDim.x, smem + ((it + 1) & 1) * STB);
    } else {
      stage_in<D, 8, SBX, NT, true>(reinterpret_cast<const char *>(x) + e0 * MBX, sx, cnt, tid);
      stage_in<D, 8, SBX, NT, true>(reinterpret_cast<const char *>(y) + e0 * MBX, sy, cnt, tid);
      stage_in<Q, 8, SBQ, NT, true>(reinterpret_cast<const char *>(op) + e0 * MBQ, so, cnt, tid);
      __syncthreads();
    }
    if (tid < cnt) {
      const double *X = reinterpret_cast<const double *>(sx + tid * SBX);
      const double *O = reinterpret_cast<const double *>(so + tid * SBQ);
      double *Y = reinterpret_cast<double *>(sy + tid * SBX);
      double S[Q][Q];
#pragma unroll
      for (int a = 0; a < Q; ++a)
#pragma unroll
        for (int b = 0; b < Q; ++b) S[a][b] = 0.0;
      // to quadrature points: contract dx, then dy (Laghos order)
#pragma unroll
      for (int dy = 0; dy < D; ++dy) {
        double sol_x[Q];
#pragma unroll
        for (int qx = 0; qx < Q; ++qx) sol_x[qx] = 0.0;
#pragma unroll
        for (int dx = 0; dx < D; ++dx) {
          const double s = X[dy * D + dx];
#pragma unroll
          for (int qx = 0; qx < Q; ++qx) sol_x[qx] = fmaT(sB[qx * D + dx], s, sol_x[qx]);
        }
#pragma unroll
        for (int qy = 0; qy < Q; ++qy) {
          const double d2q = sB[qy * D + dy];
#pragma unroll
          for (int qx = 0; qx < Q; ++qx) S[qy][qx] = fmaT(d2q, sol_x[qx], S[qy][qx]);
        }
      }
#pragma unroll
      for (int qy = 0; qy < Q; ++qy)
#pragma unroll
        for (int qx = 0; qx < Q; ++qx) S[qy][qx] *= O[qy * Q + qx];
      // back to dofs: contract qx, then qy; accumulate into the staged y
#pragma unroll
      for (int qy = 0; qy < Q; ++qy) {
        double sol_x[D];
#pragma unroll
        for (int dx = 0; dx < D; ++dx) sol_x[dx] = 0.0;
#pragma unroll
        for (int qx = 0; qx < Q; ++qx) {
          const double s = S[qy][qx];
#pragma unroll
          for (int dx = 0; dx < D; ++dx) sol_x[dx] = fmaT(sB[qx * D + dx], s, sol_x[dx]);
        }
#pragma unroll
        for (int dy = 0; dy < D; ++dy) {
          const double q2d = sB[qy * D + dy];
#pragma unroll
          for (int dx = 0; dx < D; ++dx) Y[dy * D + dx] = fmaT(q2d, sol_x[dx], Y[dy * D + dx]);
        }
      }
    }
    __syncthreads();
    stage_out<D, 8, SBX, NT, true>(reinterpret_cast<char *>(y) + e0 * MBX, sy, cnt, tid);
    if constexpr (!PF) __syncthreads();
  }
}

// ----------------------------------------------------------------------
// DMMA variant (r02; jm_plan.h mass_dmma): one WARP per element, the four
// contractions as FP64 tensor-core products (DMMA.8x8x4, D and Q padded to 8),
// no shared memory.  With lane (r = lane/4, j = lane%4) and the k-step s
// summing over k = 2j + s, an accumulator fragment (lane holds M[r][2j+e])
// is, with no data movement, both the A operand of M.C and the B operand of
// C.M^T.  Written that way, the chain is
//     M1 = B . X^T          (X^T as the B operand: lane loads X[r][2j..2j+1], 16 B)
//     M2 = M1 . B^T = S^T   (S = B X B^T; lane holds S[2j+e][r])
//     G^T = S^T .* op^T     (lane loads op[2j+e][r])
//     M3 = B^T . G          (G^T's fragment is G as the B operand)
//     Y += M3 . B           (Y itself is the accumulator: 16-B load and store)
// = Y + B^T ((B X B^T) .* op) B, with two constant fragments per lane:
// F1[s] = B[r][2j+s] (A of step 1, B operand of step 2) and F2[s] = B[2j+s][r]
// (A of step 3, B operand of step 4).  8 DMMA per element = exactly the
// 4DQ(D+Q) flops at D = Q = 8.  The thread-per-element kernel above issues one
// broadcast shared load of B per FMA and was LDS-bound (0.29 of HBM at
// D = Q = 8, profiles/r01_mass_f7_analog.jsonl).  Each warp keeps the next
// element's x / y / op loads in flight while it computes the current one.
template <int D, int Q>
__device__ __forceinline__ void mass_dmma_body(const double *__restrict__ B, const double *__restrict__ op,
                                               const double *__restrict__ x, double *__restrict__ y,
                                               long long elements) {
  constexpr int WPC = MASS_DMMA_THREADS / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, r = lane >> 2, j = lane & 3;
  double F1[2], F2[2];
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const int k = 2 * j + s;
    F1[s] = (r < Q && k < D) ? B[r * D + k] : 0.0;
    F2[s] = (k < Q && r < D) ? B[k * D + r] : 0.0;
  }
  // Each lane copies exactly the entries it will own as fragments (even D:
  // its x / y pair as one 16-B cp.async; out-of-range entries zero-filled)
  // into its own bytes of the warp's slot, so no barrier is needed: PD slots
  // per warp keep PD elements' loads in flight without holding registers.
  // Slot: x at lane*16, y at 512 + lane*16, op at 1024 + lane*16.
  constexpr int PD = JM_MASS_DMMA_PD;
  extern __shared__ __align__(16) char smem[];
  char *const wbase = smem + warp * (PD * MASS_DMMA_SLOT) + lane * 16;
  const bool okp = r < D && 2 * j < D, ok1 = r < D && 2 * j + 1 < D;
  const bool oq0 = 2 * j < Q && r < Q, oq1 = 2 * j + 1 < Q && r < Q;
  auto issue = [&](long long e, int slot) {
    if (e < elements) {
      const double *xe = x + e * (D * D), *ye = y + e * (D * D), *oe = op + e * (Q * Q);
      char *sl = wbase + slot * MASS_DMMA_SLOT;
      if constexpr (D % 2 == 0) {
        cp_async_zfill16(sl, okp ? xe + r * D + 2 * j : x, okp ? 16 : 0);
        cp_async_zfill16(sl + 512, okp ? ye + r * D + 2 * j : y, okp ? 16 : 0);
      } else {
        cp_async_zfill8(sl, okp ? xe + r * D + 2 * j : x, okp ? 8 : 0);
        cp_async_zfill8(sl + 8, ok1 ? xe + r * D + 2 * j + 1 : x, ok1 ? 8 : 0);
        cp_async_zfill8(sl + 512, okp ? ye + r * D + 2 * j : y, okp ? 8 : 0);
        cp_async_zfill8(sl + 520, ok1 ? ye + r * D + 2 * j + 1 : y, ok1 ? 8 : 0);
      }
      cp_async_zfill8(sl + 1024, oq0 ? oe + (2 * j) * Q + r : op, oq0 ? 8 : 0);
      cp_async_zfill8(sl + 1032, oq1 ? oe + (2 * j + 1) * Q + r : op, oq1 ? 8 : 0);
    }
    cp_async_commit();   // (an empty group past the end keeps the group count uniform)
  };
  const long long nw = (long long)gridDim.x * WPC;
  long long e = (long long)blockIdx.x * WPC + warp;
#pragma unroll
  for (int q = 0; q < PD; ++q) issue(e + q * nw, q);
  int slot = 0;
  for (; e < elements; e += nw) {
    cp_async_wait_group<PD - 1>();   // this lane's copies of element e have landed
    const char *sl = wbase + slot * MASS_DMMA_SLOT;
    const double2 xv = *reinterpret_cast<const double2 *>(sl);
    const double2 yv = *reinterpret_cast<const double2 *>(sl + 512);
    const double2 ov = *reinterpret_cast<const double2 *>(sl + 1024);
    double m0 = 0.0, m1 = 0.0, s0 = 0.0, s1 = 0.0;
    dmma884(m0, m1, F1[0], xv.x);    // M1 = B . X^T
    dmma884(m0, m1, F1[1], xv.y);
    dmma884(s0, s1, m0, F1[0]);      // M2 = M1 . B^T = S^T
    dmma884(s0, s1, m1, F1[1]);
    s0 *= ov.x;                      // G^T = S^T .* op^T
    s1 *= ov.y;
    m0 = 0.0; m1 = 0.0;
    dmma884(m0, m1, F2[0], s0);      // M3 = B^T . G
    dmma884(m0, m1, F2[1], s1);
    double y0 = yv.x, y1 = yv.y;
    dmma884(y0, y1, m0, F2[0]);      // Y += M3 . B
    dmma884(y0, y1, m1, F2[1]);
    double *ye = y + e * (D * D);
    if constexpr (D % 2 == 0) {
      if (okp) __stcs(reinterpret_cast<double2 *>(ye + r * D + 2 * j), make_double2(y0, y1));
    } else {
      if (okp) ye[r * D + 2 * j] = y0;
      if (ok1) ye[r * D + 2 * j + 1] = y1;
    }
    issue(e + PD * nw, slot);        // the slot's values are consumed: refill it
    slot = slot + 1 == PD ? 0 : slot + 1;
  }
  cp_async_wait_group<0>();
}

template <int D, int Q>
__global__ void __launch_bounds__(plan_mass(D, Q).threads, mass_dmma(D, Q) ? JM_MASS_DMMA_MINB : 1)
    k_mass(const double *__restrict__ B, const double *__restrict__ op, const double *__restrict__ x,
           double *__restrict__ y, long long elements) {
  static_assert(D >= 1 && D <= MASS_MAX && Q >= 1 && Q <= MASS_MAX, "1 <= D, Q <= 8");
  if constexpr (mass_dmma(D, Q)) mass_dmma_body<D, Q>(B, op, x, y, elements);
  else mass_body<D, Q>(B, op, x, y, elements);
}

}  // namespace jm
#endif  // JM_MASS_CUH
