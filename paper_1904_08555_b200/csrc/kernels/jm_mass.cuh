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
// kernel is a streaming one: one thread per element, x / op / y chunks staged
// through shared memory with coalesced 128-bit copies at an odd 16-B stride
// (conflict-free per-thread reads), B in shared memory (broadcast reads), the
// quadrature-point values S in registers.  Appended to the NVRTC source.
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
  extern __shared__ __align__(16) char smem[];
  char *sx = smem;
  char *sy = sx + stage_bytes(MPC, D, 8);
  char *so = sy + stage_bytes(MPC, D, 8);
  double *sB = reinterpret_cast<double *>(so + stage_bytes(MPC, Q, 8));
  const int tid = threadIdx.x;
  for (int i = tid; i < Q * D; i += NT) sB[i] = B[i];
  const long long nchunks = (elements + MPC - 1) / MPC;
  for (long long ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
    const long long e0 = ch * MPC;
    const int cnt = (int)((elements - e0) < MPC ? (elements - e0) : MPC);
    stage_in<D, 8, SBX, NT, true>(reinterpret_cast<const char *>(x) + e0 * MBX, sx, cnt, tid);
    stage_in<D, 8, SBX, NT, true>(reinterpret_cast<const char *>(y) + e0 * MBX, sy, cnt, tid);
    stage_in<Q, 8, SBQ, NT, true>(reinterpret_cast<const char *>(op) + e0 * MBQ, so, cnt, tid);
    __syncthreads();
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
    __syncthreads();
  }
}

template <int D, int Q>
__global__ void __launch_bounds__(MASS_THREADS)
    k_mass(const double *__restrict__ B, const double *__restrict__ op, const double *__restrict__ x,
           double *__restrict__ y, long long elements) {
  static_assert(D >= 1 && D <= MASS_MAX && Q >= 1 && Q <= MASS_MAX, "1 <= D, Q <= 8");
  mass_body<D, Q>(B, op, x, y, elements);
}

}  // namespace jm
#endif  // JM_MASS_CUH
