// jm_plan.h — launch/tiling plan shared by the host runtime (g++) and the
// device kernels (nvcc and NVRTC).  Pure constexpr C++: no CUDA, no std headers
// (NVRTC compiles it from the in-library source string).
//
// The plan picks, per (N, dtype), how a batch of independent N x N matrices is
// mapped onto the B200:
//   TPM   thread-per-matrix, whole matrix in registers      f64 N<=7, f32 N<=11
//   DMMA  FP64 tensor-core DMMA.8x8x4 (mma.sync m8n8k4.f64), N padded to 8k;
//         W warps per matrix (W=1 up to N=40 resident / 32 streaming, else a CTA)
//   F32   FP32 register-tiled outer products with FFMA2, W warps per matrix
//   GENERIC the AoT runtime-N kernel (never NVRTC-compiled)
#ifndef JM_PLAN_H
#define JM_PLAN_H

#if defined(__CUDACC__) || defined(__CUDACC_RTC__)
#define JM_HD __host__ __device__
#else
#define JM_HD
#endif

namespace jm {

enum class Addend : int { Ones = 0, Identity = 1 };
enum class Tile : int { Generic = 0, TPM = 1, Dmma = 2, Tpm2 = 3 /* r01, removed */, F32 = 4, Tpms = 5,
                        Rows = 6 /* r01 FP64 row panels, removed */,
                        F32Rows = 7 /* plan label only: the FP32 row panels of Tile::F32 */,
                        Reg = 8 /* FP64 register tiles (DFMA; run_f64t) */,
                        Lat = 9 /* latency path: a warp per matrix, an element per lane (k_update_lat) */,
                        F32Tc = 10 /* plan label only: the FP32 kind on the tensor cores (run_f32tc) */ };

struct Plan {
  int tile;      // Tile
  int threads;   // threads per CTA
  int mpc;       // matrices per CTA chunk
  int smem;      // dynamic shared memory bytes per CTA
  int w;         // warps cooperating on one matrix
};

JM_HD constexpr int cdiv(int a, int b) { return (a + b - 1) / b; }
JM_HD constexpr int rup(int a, int b) { return cdiv(a, b) * b; }

// Bytes per matrix in a shared-memory staging area.  When the matrix is a
// multiple of 16 B the stride is an ODD multiple of 16 B, so a thread-per-matrix
// read of 16-B pieces is bank-conflict free; otherwise (odd N) the matrices are
// packed and element reads at an odd element stride are conflict free.
JM_HD constexpr int stage_stride(int n, int es) {
  return ((n * n * es) % 16) ? n * n * es
                             : ((((n * n * es) / 16) & 1) ? n * n * es : n * n * es + 16);
}

// A chunk's staging area, rounded to 16 B so the buffers after it stay aligned.
JM_HD constexpr int stage_bytes(int mpc, int n, int es) { return rup(mpc * stage_stride(n, es), 16); }

// FP64: thread-per-matrix up to n = 7 (166 registers, no spill; DMMA would pad
// 7 -> 8), FP64 tensor cores above.  Measured and removed in r02 (the source
// NVRTC parses for every key keeps only kinds that ship): FP64 DFMA row
// panels for n = 9..12 (0.26-0.35 of the FP64 pipe, shared-memory operand
// bound; profiles/r01_f64_rows_g2_g4.txt) and a two-thread-per-matrix DFMA
// kind for n = 8 (0.71 vs the warp DMMA tile's 0.83; profiles/r01_tpm2_n8.jsonl).
// FP64 n = 8: the warp DMMA tile reaches 0.83 of the FP64 pipe, 0.90 of its
// bare DMMA + DFMA mix (0.92, tools/microbench k_mix2_2; the rest is the
// per-update publish / fragment loads / syncs).
// FP32: thread per matrix up to n = 11 (m and p: 242 floats, 216 registers,
// no spill).  n = 9..11 ran on the row panels at 0.28-0.43 of the FP32 pipe
// (R = 100; padding to 4-column chunks and 3-row panels); thread per matrix
// with prefetching stage reaches 0.79-0.82, and 0.86-0.93 of HBM at R = 1
// (profiles/r01_f32_tpm_n9_11.jsonl).  n = 12 (288 floats) would spill.
#ifndef JM_F32_TPM_MAX
#define JM_F32_TPM_MAX 11
#endif
// FP64 n = 9, 10: thread per matrix with the product staged row by row in the
// matrix's own shared-memory slot (Tile::Tpms, run_tpms): M stays in registers
// (81 / 100 doubles), P (which needs the old M until its last row) waits in the
// slot.  DMMA pads these sizes to 16 x 16 tiles (0.23 of the pipe).
// FP32 n = 12..14: thread per matrix with the product staged in the slot
// (run_tpms, FFMA2 rows): 0.70 of the FP32 pipe at R = 100 against 0.48-0.60
// for the row panels (n = 13: 0.44 -> 0.70); n = 15 (255 registers) is slower
// than the row panels and keeps them (profiles/r01_f32_tpms.jsonl)
#ifndef JM_F32_TPMS_MAX
#define JM_F32_TPMS_MAX 14
#endif
#ifndef JM_TPMS_ROWS
#define JM_TPMS_ROWS 1               // rows of P formed between scheduling fences (run_tpms)
#endif
#ifndef JM_F64_TPMS_MAX
#define JM_F64_TPMS_MAX 10
#endif
JM_HD constexpr bool f64t_use(int n);
JM_HD constexpr Tile tile_for(int n, int dtype) {
  return dtype == 1 ? (n <= 7 ? Tile::TPM
                       : f64t_use(n) ? Tile::Reg
                       : (n >= 9 && n <= JM_F64_TPMS_MAX) ? Tile::Tpms
                       : Tile::Dmma)
                    : (n <= JM_F32_TPM_MAX ? Tile::TPM
                       : (n <= JM_F32_TPMS_MAX ? Tile::Tpms : Tile::F32));
}

// ---- TPM ----
constexpr int TPM_THREADS = 128;

// ---- DMMA (FP64) ----
#ifndef JM_DMMA_WARP_MAX
#define JM_DMMA_WARP_MAX 40          // resident kernel: whole matrix in one warp up to this n
#endif
#ifndef JM_DMMA_WARP_MAX_STREAM
#define JM_DMMA_WARP_MAX_STREAM 32   // streaming variant: whole matrix in one warp up to this n
#endif
#ifndef JM_DMMA_RT_T8_7
#define JM_DMMA_RT_T8_7 1            // resident n = 49..56: row tiles per warp (4 = two warps of 4 + 3)
#endif
#ifndef JM_DMMA_RT_LARGE
#define JM_DMMA_RT_LARGE 1   // row tiles per warp for other n > WARP_MAX (one warp per 8-row tile)
#endif
// (r02: the border generalised to BR = 3, 4 — two-chunk column loads,
// reduce-scatter shuffles — measured slower than the padded tiles with
// k-compaction: n = 19 0.54 -> 0.45, 20 0.64 -> 0.49, 28 0.72 -> 0.60,
// 36 0.76 -> 0.69 of the FP64 pipe at R = 100; profiles/r02_ab_dmma.md)
#ifndef JM_DMMA_BORDER_MAX
#define JM_DMMA_BORDER_MAX 2         // n = 8K + r, r <= this: border tiles by DFMA (run_dmma BORD)
#endif
#ifndef JM_DMMA_BORDER_MIN
#define JM_DMMA_BORDER_MIN 16        // ... and n above this
#endif
// k-compaction (run_dmma CMP): n = 8K + r with 2 <= r <= 4 puts the last k
// tile's r real k into ONE k-step (k = 8K + t) instead of the two half-padding
// k-steps of the k-permutation; its A fragment takes two shuffles per row tile
#ifndef JM_DMMA_KCOMPACT
#define JM_DMMA_KCOMPACT 1
#endif
constexpr int DMMA_WPC = 4;                       // warps per CTA when W == 1
JM_HD constexpr int dmma_t8(int n) { return cdiv(n, 8); }
// Row tiles per warp (W = T8 / RT warps share a matrix), measured on B200
// (profiles/r01_dmma_rt_sweep.jsonl, FP64 pipe fraction at R = 100):
//  * whole matrix per warp (RT = T8) up to n = 40 in the resident kernel:
//    n = 33..40 0.51-0.82 -> 0.60-0.93 over one warp per 8-row tile, the
//    B fragment of a k-step now feeding 5 row tiles instead of 1 (210-226
//    registers, 2 CTAs of 4 warps per SM, no spill);
//  * 41..48 (T8 = 6): two warps of 3 row tiles (n = 48 0.84 -> 0.93, n = 44
//    0.65 -> 0.70; up to 255 registers, no spill);
//  * 57..64 (T8 = 8): four warps of 2 row tiles (n = 64 0.96);
//  * 49..56 (T8 = 7): one warp per row tile.  Two warps of 4 + 3 row tiles
//    (JM_DMMA_RT_T8_7=4, RAG in run_dmma) measured worse: 255 registers,
//    8 warps per SM, n = 49 0.61 -> 0.43, n = 56 0.82 -> 0.70
//    (profiles/r01_dmma_rt_experiments.jsonl).
// The streaming variant keeps one warp per row tile above n = 32: its ring
// leaves too little shared memory for 4 whole-matrix warps per CTA, and at
// its low repeat counts the wider CTAs stream better.
JM_HD constexpr int dmma_rt(int n, bool strm = false) {
  return n <= (strm ? JM_DMMA_WARP_MAX_STREAM : JM_DMMA_WARP_MAX) ? dmma_t8(n)
         : dmma_t8(n) == 8                                         ? 2
         : (!strm && dmma_t8(n) == 6)                              ? 3
         : (!strm && dmma_t8(n) == 7)                              ? JM_DMMA_RT_T8_7
                                                                   : JM_DMMA_RT_LARGE;
}
JM_HD constexpr int dmma_w(int n, bool strm = false) { return cdiv(dmma_t8(n), dmma_rt(n, strm)); }
JM_HD constexpr int dmma_rsc(int n) { return rup(4 * dmma_t8(n), 8); }     // scratch row stride, 16-B chunks
JM_HD constexpr int dmma_scr(int n) { return 8 * dmma_t8(n) * dmma_rsc(n) * 16; }  // one scratch buffer

// ---- F32 tiles, r02 ("F32T", run_f32t) ----
// r01's tiles (8 x 16 blocks, ~230-255 registers, 2-way conflicted shared
// loads) kept the FMA pipe 55-73 % busy (profiles/r02_ncu_baseline.md).
// run_f32t keeps the algorithm (thread-owned RA x CB blocks of P, the A
// operand by LDS.128 of M[row][k..k+3], each row's block reloaded right after
// its last use, the B operand by LDS.128 of row k one k ahead) and chooses,
// per n, the register tile, the shared-memory layout, a register cap and the
// unrolling of the k loop.  What bounds it (profiles/r02_f32_microbench.md):
// * shared-memory wavefronts: an LDS.128 runs as two half-warps; a half costs
//   one wavefront when its two quarter-warps touch disjoint 16-B bank slots
//   (or one address), else the sum of the quarters (tools/microbench/
//   lds_wavefronts.cu under ncu).  The layouts below are conflict free under
//   that rule (tools/f32_layout.py; ncu: 0-2 % conflicts);
// * the register-file return of shared loads: a pure FFMA2 stream runs at
//   0.97 of the FP32 pipe, with one LDS.128 per 16 FFMA2 at 0.91, with two
//   at 0.77-0.81 (tools/microbench/ffma2_lds_mix.cu) — so bigger register
//   tiles (fewer loaded registers per FFMA2) win even at two warps per SMSP.
// Lane packing (r02 late, F32T.pack): a matrix of RG*CG threads that does not
// divide 32 leaves lanes idle in a warp-per-matrices mapping (9 x 6 FP64
// tiles: 6 threads, 5 matrices, 2 of 32 lanes idle; 28-thread FP32 tiles: 4
// of 32).  Packed, thread tid of the CTA is thread tid % (RG*CG) of matrix
// tid / (RG*CG), and a CTA of WPC warps holds 32*WPC / (RG*CG) matrices; the
// per-update syncs become CTA barriers.  JM_TILE_PACK=0: off everywhere;
// JM_TILE_PACK_N / _DT / _WPC: force it for one size (measurement hook).
#ifndef JM_TILE_PACK
#define JM_TILE_PACK 1
#endif
#ifndef JM_TILE_PACK_N
#define JM_TILE_PACK_N 0
#endif
#ifndef JM_TILE_PACK_DT
#define JM_TILE_PACK_DT 1
#endif
#ifndef JM_TILE_PACK_WPC
#define JM_TILE_PACK_WPC 0
#endif
// JM_TILE_PACK_ALL (measurement hook): pack every resident tile shape that
// idles lanes, with the smallest (1) or the largest (2) CTA of <= 8 warps
// that the packing fills
#ifndef JM_TILE_PACK_ALL
#define JM_TILE_PACK_ALL 0
#endif
#ifndef JM_TILE_PACK_STRM
#define JM_TILE_PACK_STRM 0   // 1: JM_TILE_PACK_ALL also packs the low-repeat kernels' shapes
#endif
JM_HD constexpr int pack_fill_milli(int tpm, int w) { return (32 * w / tpm) * tpm * 1000 / (32 * w); }
JM_HD constexpr int unpacked_fill_milli(int tpm) {
  return tpm > 32 ? tpm * 1000 / (32 * ((tpm + 31) / 32)) : (32 / tpm) * tpm * 1000 / 32;
}
JM_HD constexpr int pack_wpc_for(int tpm, int mode) {
  int best = 0;
  for (int w = 2; w <= 8; ++w)
    if (32 * w >= tpm && pack_fill_milli(tpm, w) >= 990 && (best == 0 || mode == 2)) best = w;
  return best;
}
struct F32T {
  int ra, cb, rg, cg;   // RA x CB register tile; RG x CG threads per matrix
  int ldm;              // row stride of the published M, floats (multiple of 4)
  int pad;              // extra 16-B chunks per matrix region (bank-slot offset between matrices)
  int colblk;           // 1: thread column tc owns chunks tc*CB/4 + h (blocked), 0: h*CG + tc
  int trfast;           // 1: thread t of a matrix is (tr, tc) = (t % RG, t / RG), 0: (t / CG, t % CG)
  int qmix;             // 1 (two matrices per warp): quarter-warp q holds matrix q % 2
  int maxreg;           // register cap (__maxnreg__ of k_update_rc)
  int kunroll;          // k blocks of four per iteration of the (rolled) k loop
  int wpc;              // warps per CTA
  int pack;             // 1: lane-packed CTA (matrices of RG*CG threads laid end to end over
                        // the CTA's threads, straddling warps; a CTA barrier per sync)
};
// Per-n choices, measured on B200 (tools/f32_search.py; the layout of each
// shape from tools/f32_layout.py):
// {n, RA, CB, row padding (16-B chunks), region padding (16-B chunks), colblk, trfast, qmix, maxreg, kunroll}
struct F32TRow { int n, ra, cb, ldmpad, pad, colblk, trfast, qmix, maxreg, kunroll, wpc, pack; };   // (wpc 0: 4)
// FP64 register tiles (DFMA, run_f64t) for the sizes where DMMA's 8 x 8 x 4
// granularity wastes most of the pipe; the same fields, CB a multiple of 2
// (a 16-B chunk holds two doubles).  Only the sizes listed take this kind.
// Picked from the r02 search (tools/f64_candidates.json, profiles/r02_f64_search.jsonl)
// and kept where they beat the DMMA tile WITH k-compaction (profiles/r02_ab_dmma.md,
// FP64 pipe at R = 100, DMMA in brackets): n = 11 0.512 (0.375), 12 0.636 (0.496),
// 17 0.553 (0.536), 18 0.628 (0.480), 19 0.613 (0.542), 20 0.704 (0.636) — 17
// and 18 as 9 x 6 tiles from the wider search (profiles/r02_f64_wide_search.jsonl);
// n = 35 (0.656 vs 0.689)
// stays DMMA.  Their low-repeat kernel is the DMMA ring (plan_stream).
// JM_F64T_ON=0: none.
#ifndef JM_F64T_ON
#define JM_F64T_ON 1
#endif
constexpr F32TRow F64T_TABLE[] = {
    {0, 0, 0, 0, 0, 0, 0, 0, 0, 0},
#if JM_F64T_ON
    {11, 3, 12, 4, 1, 0, 1, 0, 255, 2},
    {12, 3, 12, 4, 1, 0, 1, 0, 168, 6},
    {17, 9, 6, 3, 1, 1, 1, 0, 168, 8},    // (r02 wide search: 0.553 vs the border DMMA's 0.536; cap 168: 0.555)
    {18, 9, 6, 3, 1, 1, 1, 0, 200, 9},    // (r02 wide search: 0.628, cap 200: 0.638; 6 x 10 0.560)
    {19, 5, 10, 4, 1, 1, 1, 0, 168, 9},   // (cap 168: 0.615)
    {20, 5, 10, 4, 1, 1, 1, 0, 168, 10},  // (cap 168: 0.712)
#endif
};
constexpr F32TRow F32T_TABLE[] = {
    {16, 4, 16, 2, 1, 0, 1, 0, 168, 4},  // 0.721 of the pipe, 148 regs (row panels 0.708)
    {17, 6, 20, 2, 1, 0, 1, 0, 255, 4},  // 0.515 of the pipe, 200 regs (r02 wide search; was 0.434)
    {18, 6, 20, 2, 1, 0, 1, 0, 255, 4},  // 0.586 of the pipe, 247 regs (r02 wide search; was 0.491)
    {19, 5, 20, 1, 1, 0, 1, 0, 255, 4},  // 0.638 of the pipe, 205 regs (r02 wide search; was 0.487)
    {20, 5, 12, 4, 1, 1, 1, 0, 168, 5},  // 0.618 of the pipe, 146 regs
    {21, 11, 12, 1, 2, 0, 1, 0, 255, 5, 2},  // 0.574 of the pipe, 220 regs (r02 wpc search; was 0.562)
    {22, 6, 12, 4, 1, 1, 1, 0, 168, 5},  // 0.609 of the pipe, 150 regs
    {23, 6, 12, 4, 1, 1, 1, 0, 168, 5},  // 0.654 of the pipe, 154 regs
    {24, 6, 12, 4, 1, 1, 1, 0, 168, 6},  // 0.721 of the pipe, 158 regs
    {25, 5, 16, 1, 1, 1, 0, 0, 168, 6},  // 0.543 of the pipe, 152 regs
    {26, 7, 8, 1, 1, 1, 0, 1, 168, 6},  // 0.569 of the pipe, 148 regs
    {27, 7, 8, 1, 1, 1, 0, 1, 168, 6},  // 0.599 of the pipe, 140 regs
    {28, 7, 8, 1, 1, 1, 0, 1, 168, 7},  // 0.660 of the pipe, 148 regs
    {29, 8, 8, 1, 3, 1, 0, 1, 168, 7},  // 0.615 of the pipe, 148 regs
    {30, 8, 8, 1, 3, 1, 0, 1, 168, 7},  // 0.668 of the pipe, 152 regs
    {31, 4, 16, 2, 3, 0, 0, 1, 168, 7},  // 0.700 of the pipe, 148 regs
    {32, 4, 16, 2, 3, 0, 0, 1, 168, 8},  // 0.756 of the pipe, 142 regs
    {33, 7, 12, 1, 1, 1, 0, 1, 168, 8},  // 0.575 of the pipe, 152 regs
    {34, 7, 12, 1, 1, 1, 0, 1, 168, 8},  // 0.636 of the pipe, 161 regs
    {35, 7, 12, 1, 1, 1, 0, 1, 168, 8},  // 0.662 of the pipe, 156 regs
    {36, 8, 12, 1, 1, 1, 0, 1, 255, 9},  // 0.595 of the pipe, 200 regs
    {37, 5, 20, 1, 0, 0, 1, 0, 232, 4},  // 0.626 of the pipe (r02 neighbourhood search: cap 232, k unroll 4; was 0.585)
    {38, 5, 12, 1, 0, 0, 1, 0, 168, 9},  // 0.584 of the pipe, 144 regs
    {39, 5, 12, 1, 0, 0, 1, 0, 168, 9},  // 0.613 of the pipe, 134 regs
    {40, 5, 12, 1, 0, 0, 1, 0, 168, 10},  // 0.656 of the pipe, 142 regs
    {41, 6, 12, 1, 0, 0, 0, 0, 168, 10},  // 0.554 of the pipe, 154 regs
    {42, 6, 12, 1, 0, 0, 0, 0, 168, 10},  // 0.611 of the pipe, 153 regs
    {43, 6, 12, 1, 0, 0, 1, 0, 168, 10},  // 0.604 of the pipe, 156 regs
    {44, 6, 12, 1, 0, 0, 1, 0, 168, 11},  // 0.644 of the pipe, 160 regs
    {45, 6, 12, 1, 0, 0, 1, 0, 168, 11},  // 0.662 of the pipe, 148 regs
    {46, 6, 12, 1, 0, 0, 1, 0, 168, 11},  // 0.700 of the pipe, 154 regs
    {47, 6, 12, 1, 0, 0, 1, 0, 168, 4},  // 0.732 of the pipe (r02 neighbourhood search: cap 168, k unroll 4; was 0.719)
    {48, 6, 12, 1, 0, 0, 1, 0, 168, 12},  // 0.750 of the pipe, 154 regs
    {49, 13, 8, 4, 0, 0, 1, 0, 232, 4},  // 0.531 of the pipe, 212 regs (r02 neighbourhood search: cap 232, k unroll 4; wide search 0.518)
    {50, 13, 8, 4, 0, 0, 1, 0, 232, 4},  // 0.551 of the pipe, 215 regs (r02 neighbourhood search: cap 232, k unroll 4; wide search 0.534)
    {51, 13, 8, 4, 0, 0, 1, 0, 232, 4},  // 0.573 of the pipe (r02 neighbourhood search: cap 232, k unroll 4; was 0.560)
    {52, 13, 8, 1, 0, 0, 1, 0, 255, 4},  // 0.585 of the pipe, 236 regs (r02 neighbourhood search: k unroll 4; wide search 0.533)
    {53, 7, 16, 1, 0, 0, 1, 0, 232, 4},  // 0.588 of the pipe (r02 neighbourhood search: cap 232, k unroll 4; was 0.555)
    {54, 7, 8, 1, 0, 0, 1, 0, 144, 8},  // 0.618 of the pipe (r02 cap A/B, profiles/r02_ab_f32_cap.md: cap 144; cap 168 0.605)
    {55, 7, 8, 1, 0, 0, 1, 0, 144, 8},  // 0.638 of the pipe (r02 cap A/B: cap 144; cap 232 0.620)
    {56, 7, 16, 1, 0, 0, 1, 0, 255, 2},  // 0.662 of the pipe, 204 regs
    {57, 8, 16, 1, 0, 0, 1, 0, 255, 2},  // 0.587 of the pipe, 225 regs
    {58, 8, 16, 1, 0, 0, 1, 0, 255, 4},  // 0.628 of the pipe (r02 neighbourhood search: cap 255, k unroll 4; was 0.611)
    {59, 8, 8, 1, 0, 0, 0, 0, 255, 2},  // 0.640 of the pipe, 154 regs
    {60, 8, 16, 1, 0, 0, 1, 0, 232, 4},  // 0.676 of the pipe (r02 neighbourhood search: cap 232, k unroll 4; was 0.633)
    {61, 8, 16, 1, 0, 0, 1, 0, 255, 2},  // 0.679 of the pipe, 236 regs
    {62, 8, 16, 1, 0, 0, 1, 0, 255, 2},  // 0.711 of the pipe, 244 regs
    {63, 8, 16, 1, 0, 0, 1, 0, 255, 2},  // 0.730 of the pipe, 236 regs
    {64, 8, 16, 1, 0, 0, 1, 0, 255, 4},  // 0.781 of the pipe (r02 neighbourhood search: cap 255, k unroll 4; was 0.763)
};
// The low-repeat (streaming) kernel's own shapes, where they differ from the
// resident kernel's (R = 1 is bound by moving the matrices, so a smaller work
// region -- more warps per SM -- can beat the faster k loop); same fields.
constexpr F32TRow F32TS_TABLE[] = {
    {0, 0, 0, 0, 0, 0, 0, 0, 0, 0},
    // Streaming-kernel shapes, R = 1, fraction of the HBM bandwidth (bytes moved / time) of the
    // kernel the library picks ("was" = the resident shape); last field 2 = two-warp CTAs.
    // Odd n: search v2 (profiles/r02_f32_stream_search_v2.jsonl); even n: search v3 with the
    // one-time packed accesses in the layout model and PVEC on (r02_f32_stream_search_v3.jsonl);
    // n = 42, 44, 52, 54 stream fastest with their resident shape.
    {16, 8, 4, 1, 4, 0, 1, 0, 255, 2},  // 0.930 at R = 1 (r02 neighbourhood search: cap 255, k unroll 2; was 0.859)
    {17, 6, 4, 6, 0, 0, 1, 1, 168, 4, 2},  // 0.448 at R = 1 (was 0.316), 106 regs
    {18, 5, 12, 4, 2, 0, 1, 0, 255, 4, 2},  // 0.740 at R = 1 (r02 neighbourhood search: cap 255, k unroll 4; was 0.707)
    {19, 5, 12, 4, 1, 1, 1, 0, 168, 4, 2},  // 0.413 at R = 1 (was 0.386), 137 regs
    {20, 5, 12, 4, 1, 1, 1, 0, 168, 5, 2},  // 0.747 at R = 1 (v3) (was 0.705), 133 regs
    {21, 7, 12, 1, 5, 0, 0, 0, 168, 5},   // the r02 resident shape before the CTA-size search (0.40 at R = 1; the 11 x 12 two-warp tile streams at 0.31)
    {22, 6, 12, 1, 2, 0, 1, 0, 168, 5},  // 0.694 at R = 1 (v3) (was 0.428), 165 regs
    {23, 8, 12, 1, 5, 0, 0, 0, 255, 5, 2},  // 0.433 at R = 1 (was 0.365), 221 regs
    {24, 6, 12, 1, 4, 1, 1, 0, 168, 6},  // 0.723 at R = 1 (v3) (was 0.506), 159 regs
    {25, 7, 8, 1, 1, 1, 0, 1, 168, 6, 2},  // 0.424 at R = 1 (was 0.365), 132 regs
    {26, 7, 8, 1, 1, 1, 0, 1, 168, 6, 2},  // 0.650 at R = 1 (v3) (was 0.618), 133 regs
    {27, 7, 8, 1, 1, 1, 0, 1, 168, 6, 2},  // 0.468 at R = 1 (was 0.455), 131 regs
    {28, 7, 8, 1, 0, 0, 0, 1, 168, 7, 2},  // 0.667 at R = 1 (v3) (was 0.628), 131 regs
    {29, 8, 8, 1, 3, 1, 0, 1, 168, 7, 2},  // 0.440 at R = 1 (was 0.428), 144 regs
    {30, 8, 8, 1, 3, 1, 0, 1, 168, 7, 2},  // 0.705 at R = 1 (v3) (was 0.667), 146 regs
    {31, 8, 8, 1, 3, 1, 0, 1, 168, 7, 2},  // 0.475 at R = 1 (was 0.428), 141 regs
    {32, 8, 8, 1, 3, 1, 0, 1, 168, 8, 2},  // 0.758 at R = 1 (v3) (was 0.681), 144 regs
    {33, 6, 8, 1, 0, 1, 1, 0, 168, 8},  // 0.351 at R = 1 (was 0.289), 122 regs
    {34, 7, 12, 2, 0, 0, 0, 1, 168, 8},  // 0.535 at R = 1 (v3) (was 0.508), 161 regs
    {35, 7, 12, 1, 1, 1, 0, 1, 168, 8, 2},  // 0.394 at R = 1 (was 0.375), 160 regs
    {36, 6, 8, 3, 0, 0, 0, 0, 168, 9},  // 0.537 at R = 1 (v3) (was 0.491), 124 regs
    {37, 7, 8, 1, 0, 1, 1, 0, 168, 9},  // 0.355 at R = 1 (was 0.334), 138 regs
    {38, 5, 12, 1, 0, 0, 1, 0, 168, 9, 2},  // 0.506 at R = 1 (v3) (was 0.485), 129 regs
    {39, 7, 8, 1, 0, 1, 1, 0, 168, 9},  // 0.376 at R = 1 (was 0.358), 137 regs
    {40, 5, 12, 1, 0, 1, 1, 0, 168, 10},  // 0.494 at R = 1 (v3) (was 0.465), 135 regs
    {46, 6, 12, 1, 0, 1, 1, 0, 168, 11},  // 0.490 at R = 1 (v3) (was 0.462), 141 regs
    {48, 6, 12, 1, 0, 1, 1, 0, 168, 12},  // 0.481 at R = 1 (v3) (was 0.396), 156 regs
    {49, 7, 16, 1, 0, 0, 0, 0, 255, 2},  // 0.258 at R = 1 (was 0.233), 214 regs
    {50, 7, 8, 1, 0, 1, 1, 0, 255, 4, 2},  // 0.380 at R = 1 (r02 neighbourhood search: cap 255, k unroll 4; was 0.364)
    {51, 7, 8, 1, 0, 0, 1, 0, 168, 2, 2},  // 0.300 at R = 1 (was 0.241), 146 regs
    {53, 7, 8, 1, 0, 0, 1, 0, 168, 2, 2},  // 0.303 at R = 1 (was 0.245), 154 regs
    {56, 7, 8, 1, 0, 0, 1, 0, 168, 8, 2},  // 0.434 at R = 1 (r02 neighbourhood search: cap 168, k unroll 8; was 0.408)
    {57, 8, 8, 1, 0, 0, 0, 0, 168, 2, 2},  // 0.303 at R = 1 (was 0.242), 146 regs
    {58, 8, 8, 1, 0, 0, 0, 0, 168, 2, 2},  // 0.410 at R = 1 (v3) (was 0.290), 154 regs
    {60, 8, 8, 1, 0, 0, 1, 0, 168, 2, 2},  // 0.414 at R = 1 (v3) (was 0.291), 146 regs
    {61, 8, 8, 1, 0, 0, 0, 0, 168, 2, 2},  // 0.324 at R = 1 (was 0.265), 150 regs
    {62, 8, 8, 1, 0, 0, 0, 0, 168, 2, 2},  // 0.428 at R = 1 (v3) (was 0.316), 152 regs
    {63, 8, 8, 1, 0, 0, 0, 0, 168, 2, 2},  // 0.295 at R = 1 (was 0.229), 153 regs
    {64, 8, 8, 1, 0, 0, 0, 0, 168, 2, 2},  // 0.459 at R = 1 (v3) (was 0.297), 155 regs
};
#ifndef JM_F32T_RA                // tuning hooks: force the register-tile shape / layout / knobs
#define JM_F32T_RA 0
#endif
#ifndef JM_F32T_CB
#define JM_F32T_CB 0
#endif
#ifndef JM_F32T_LDMPAD
#define JM_F32T_LDMPAD -1
#endif
#ifndef JM_F32T_PAD
#define JM_F32T_PAD -1
#endif
#ifndef JM_F32T_COLBLK
#define JM_F32T_COLBLK -1
#endif
#ifndef JM_F32T_TRFAST
#define JM_F32T_TRFAST -1
#endif
#ifndef JM_F32T_QMIX
#define JM_F32T_QMIX -1
#endif
#ifndef JM_F32T_MAXREG
#define JM_F32T_MAXREG 0
#endif
#ifndef JM_F32T_KUNROLL
#define JM_F32T_KUNROLL 0
#endif
#ifndef JM_F32T_WPC
#define JM_F32T_WPC 0
#endif
// the default shape when no table entry applies: the tile that covers the
// matrix with <= 64 threads and wastes least (padding x idle lanes x loads per FFMA2)
// (dt = 0 float, 1 double, 2 float in the low-repeat (streaming) kernel, which
// may take its own shape from F32TS_TABLE; VEC = 16 / element size elements
// per 16-B chunk)
JM_HD constexpr int tt_vec(int dt) { return dt == 1 ? 2 : 4; }
JM_HD constexpr int tt_es(int dt) { return dt == 1 ? 8 : 4; }
JM_HD constexpr F32T f32t_default(int n, int dt = 0) {
  const int v = tt_vec(dt), w = dt == 1 ? 2 : 1;   // elements per chunk, 32-bit registers per element
  F32T best{8, 8, cdiv(n, 8), cdiv(n, 8), 0, 0, 0, 1, 0, 168, 2, 4};
  double bs = -1.0;
  for (int ra = 8; ra >= 2; --ra)
    for (int cb = 16; cb >= v; cb -= v) {
      const int rg = cdiv(n, ra), cg = cdiv(n, cb), t = rg * cg;
      if (t > 64 || w * (ra * cb + v * ra + 2 * cb) > 200) continue;
      const double pad = (double)n * n / ((double)(rg * ra) * (cg * cb));
      const double lane = t > 32 ? (double)t / rup(t, 32) : (double)((32 / t) * t) / 32.0;
      const double core = 1.0 / (1.0 + 0.3 * 4.0 * (ra + cb) / (ra * cb));
      const double sc = pad * lane * core;
      if (sc > bs + 1e-9) { bs = sc; best = F32T{ra, cb, rg, cg, 0, 0, 0, 1, 0, 168, 2, 4, 0}; }
    }
  best.ldm = best.cg * best.cb + v;
  best.maxreg = w * (best.ra * best.cb + v * best.ra + 2 * best.cb) + 24 > 168 ? 255 : 168;
  return best;
}
JM_HD constexpr F32T f32t_tile(int n, int dt = 0) {
  F32T t = f32t_default(n, dt);
  auto take = [&](const F32TRow &r) {
    t = F32T{r.ra, r.cb, cdiv(n, r.ra), cdiv(n, r.cb), cdiv(n, r.cb) * r.cb + tt_vec(dt) * r.ldmpad, r.pad,
             r.colblk, r.trfast, r.qmix, r.maxreg, r.kunroll, r.wpc > 0 ? r.wpc : 4, r.pack};
  };
  if (dt == 1) {
    for (const F32TRow &r : F64T_TABLE)
      if (r.n == n && r.ra > 0) take(r);
  } else {
    for (const F32TRow &r : F32T_TABLE)
      if (r.n == n && r.ra > 0) take(r);
    if (dt == 2)
      for (const F32TRow &r : F32TS_TABLE)
        if (r.n == n && r.ra > 0) take(r);
  }
  if (JM_TILE_PACK == 0) t.pack = 0;
  if (JM_TILE_PACK_N == n && (dt == 1) == (JM_TILE_PACK_DT == 1) && dt != 2) {   // (search hook)
    t.pack = 1;
    if (JM_TILE_PACK_WPC > 0) t.wpc = JM_TILE_PACK_WPC;
  }
  if (JM_TILE_PACK_ALL > 0 && (dt != 2 || JM_TILE_PACK_STRM) && !t.qmix) {
    const int tpm = t.rg * t.cg, w = pack_wpc_for(tpm, JM_TILE_PACK_ALL);
    if (w > 0 && pack_fill_milli(tpm, w) > unpacked_fill_milli(tpm) + 20) { t.pack = 1; t.wpc = w; }
  }
  if (t.pack) t.qmix = 0;
  if (dt == 1) {   // (the JM_F32T_* tuning hooks below apply to the FP32 tiles)
    if (t.rg * t.cg > 16 || t.rg * t.cg <= 8) t.qmix = 0;
    return t;
  }
  if (JM_F32T_RA > 0 && JM_F32T_CB > 0) {
    t.ra = JM_F32T_RA; t.cb = JM_F32T_CB; t.rg = cdiv(n, t.ra); t.cg = cdiv(n, t.cb);
    t.ldm = t.cg * t.cb + 4;
  }
  if (JM_F32T_LDMPAD >= 0) t.ldm = t.cg * t.cb + 4 * JM_F32T_LDMPAD;
  if (JM_F32T_PAD >= 0) t.pad = JM_F32T_PAD;
  if (JM_F32T_COLBLK >= 0) t.colblk = JM_F32T_COLBLK;
  if (JM_F32T_TRFAST >= 0) t.trfast = JM_F32T_TRFAST;
  if (JM_F32T_QMIX >= 0) t.qmix = JM_F32T_QMIX;
  if (JM_F32T_MAXREG > 0) t.maxreg = JM_F32T_MAXREG;
  if (JM_F32T_KUNROLL > 0) t.kunroll = JM_F32T_KUNROLL;
  if (JM_F32T_WPC > 0) t.wpc = JM_F32T_WPC;
  if (t.rg * t.cg > 16 || t.rg * t.cg <= 8) t.qmix = 0;   // quarter mixing needs exactly two matrices per warp
  return t;
}
JM_HD constexpr int f32t_tpmat(int n, int dt = 0) { return f32t_tile(n, dt).rg * f32t_tile(n, dt).cg; }   // threads per matrix
// (a matrix of more than 32 threads takes whole warps; threads past RG*CG idle)
JM_HD constexpr int f32t_wpm(int n, int dt = 0) {   // warps per matrix
  return f32t_tpmat(n, dt) > 32 ? cdiv(f32t_tpmat(n, dt), 32) : 1;
}
JM_HD constexpr int f32t_mpw(int n, int dt = 0) {   // matrices per warp (1 for a multi-warp matrix; 2 under qmix)
  return f32t_tpmat(n, dt) > 32 ? 1 : f32t_tile(n, dt).qmix ? 2 : 32 / f32t_tpmat(n, dt);
}
JM_HD constexpr int f32t_wpc(int n, int dt = 0) {
  return f32t_tile(n, dt).wpc < f32t_wpm(n, dt) ? f32t_wpm(n, dt) : f32t_tile(n, dt).wpc;
}
JM_HD constexpr int f32t_mpc(int n, int dt = 0) {   // matrices per CTA
  return f32t_tile(n, dt).pack ? 32 * f32t_wpc(n, dt) / f32t_tpmat(n, dt)
                               : f32t_wpc(n, dt) / f32t_wpm(n, dt) * f32t_mpw(n, dt);
}
JM_HD constexpr int f32t_nr(int n, int dt = 0) { return f32t_tile(n, dt).rg * f32t_tile(n, dt).ra; }   // padded rows
JM_HD constexpr int f32t_kp(int n, int dt = 0) { return rup(n, tt_vec(dt)); }   // k blocks of one 16-B chunk
// M rows in the work area: the A loads of M[row][kb-block] read rows up to rup(n, VEC) (zero beyond n)
JM_HD constexpr int f32t_srows(int n, int dt = 0) {
  return f32t_nr(n, dt) > f32t_kp(n, dt) ? f32t_nr(n, dt) : f32t_kp(n, dt);
}
// one matrix region: the staged matrix (packed, n*n), then the published M
JM_HD constexpr int f32t_region(int n, int dt = 0) {
  return rup(f32t_srows(n, dt) * f32t_tile(n, dt).ldm * tt_es(dt) > n * n * tt_es(dt)
                 ? f32t_srows(n, dt) * f32t_tile(n, dt).ldm * tt_es(dt)
                 : n * n * tt_es(dt),
             16) +
         16 * f32t_tile(n, dt).pad;
}
// register cap (__maxnreg__ of k_update_rc): at ~150-210 registers ptxas keeps
// the next k step's B loads in flight; a lower cap forces earlier uses
JM_HD constexpr int f32t_maxreg(int n, int dt = 0) { return f32t_tile(n, dt).maxreg; }
JM_HD constexpr int f32t_kunroll(int n, int dt = 0) {
  return f32t_tile(n, dt).kunroll < 1 ? 1 : f32t_tile(n, dt).kunroll;
}
// FP64 sizes that take the register tiles: those listed in F64T_TABLE
JM_HD constexpr bool f64t_use(int n) {
  for (const F32TRow &r : F64T_TABLE)
    if (r.n == n && r.ra > 0) return true;
  return false;
}
JM_HD constexpr bool f32p_use(int n);
JM_HD constexpr bool f32t_use(int n) { return n > JM_F32_TPM_MAX && !f32p_use(n); }   // (resident kernel)
// The low-repeat kernel of a row-panel size may be the register tiles instead
// (their streaming shapes, F32TS_TABLE): n >= JM_F32T_STREAM_MIN.  Measured at
// R = 1 (profiles/r02_f32s_n15_16.jsonl): n = 16 as 8 x 4 tiles 0.89 of HBM
// against 0.54 for the row-panel ring; n = 15 0.58 against 0.72 (stays).
#ifndef JM_F32T_STREAM_MIN
#define JM_F32T_STREAM_MIN 16
#endif
JM_HD constexpr bool f32t_stream_use(int n) { return f32t_use(n) || (n > JM_F32_TPM_MAX && n >= JM_F32T_STREAM_MIN); }

// ---- F32 row panels (9 <= n <= 32) ----
// A thread owns RP = 4 FULL rows of M (the A operand is local); row k of M
// (the B operand) is a shared-memory broadcast.  G threads per matrix,
// 32 / G matrices per warp, P computed in `f32p_halves` column halves so the
// accumulators fit next to the 4 full rows.
constexpr int F32P_RP_MAX = 4;
constexpr int F32P_WPC = 2;                       // warps per CTA
constexpr int F32P_KSTEP = 4;                     // k steps between scheduling fences
// (n > 16 needs more than 4 x 16 resident floats next to the accumulators: spills)
// r02: n = 16 takes the register tiles (4 x 16: 0.72 of the FP32 pipe at
// R = 100 against 0.71 for the row panels; profiles/r02_f32_n16_resident_search.jsonl)
#ifndef JM_F32P_MAX
#define JM_F32P_MAX 15
#endif
JM_HD constexpr bool f32p_use(int n) { return n >= 9 && n <= JM_F32P_MAX; }
JM_HD constexpr int f32p_g(int n) { return n <= 16 ? 4 : 8; }                 // threads per matrix
JM_HD constexpr int f32p_mpw(int n) { return 32 / f32p_g(n); }                // matrices per warp
JM_HD constexpr int f32p_rp(int n) { return cdiv(n, f32p_g(n)); }             // rows per thread (<= 4)
JM_HD constexpr int f32p_ncr(int n) { return cdiv(n, 4); }                    // real 16-B chunks per row
JM_HD constexpr int f32p_ncs(int n) { return f32p_ncr(n) <= 4 ? 4 : 8; }      // stored chunks (pow2: XOR swizzle)
// column groups of (at most) two 16-B chunks: 8 accumulator columns live at a time
JM_HD constexpr int f32p_halves(int n) { return n <= 16 ? 1 : cdiv(f32p_ncr(n), 2); }
// one matrix buffer, +32 B skew: a matrix's PAIR of buffers is then an odd
// multiple of 64 B, so the two matrices sharing a quarter-warp land in
// opposite halves of the 128-B bank window
JM_HD constexpr int f32p_mbuf(int n) { return n * f32p_ncs(n) * 16 + 32; }
// stride between two matrices' buffer pairs (own two buffers): + JM_F32P_PAIR_SKEW
// bytes, so the four matrices of a half-warp reading row k (one 16-B address
// each) land in four bank slots (pair stride 132 chunks = 4 mod 8 put
// matrices 0/2 and 1/3 on one slot: 40 % of the n = 16 kernel's wavefronts
// conflicted, profiles/r02_ncu_kinds.md); the publish then pays 2-way
// Measured (profiles/r02_ab_skew.md): slower at every n = 12..16 (R = 1 n = 16
// 0.54 -> 0.51 of HBM, R = 100 0.71 -> 0.70 of the pipe) — off (0)
#ifndef JM_F32P_PAIR_SKEW
#define JM_F32P_PAIR_SKEW 0
#endif
JM_HD constexpr int f32p_pstr(int n) { return 2 * f32p_mbuf(n) + JM_F32P_PAIR_SKEW; }
// resident kernel: the matrix's stage slot, widened to a row buffer, doubles as
// the first row buffer (run_f32p INPL), one buffer less per matrix: n = 12
// 0.52 -> 0.65 and n = 14 0.50 -> 0.60 of the FP32 pipe at R = 100; n = 16
// (already register-limited to 5 CTAs per SM) measured 0.72 -> 0.69 and keeps
// two own buffers (profiles/r01_f32p_inplace.jsonl).  JM_F32P_INPLACE=0 turns
// it off.
#ifndef JM_F32P_INPLACE
#define JM_F32P_INPLACE 1
#endif
JM_HD constexpr bool f32p_inplace(int n) { return JM_F32P_INPLACE && (n * n * 4) % 16 == 0 && n < 16; }
JM_HD constexpr int f32p_slot(int n) {
  return rup(f32p_mbuf(n) > stage_stride(n, 4) ? f32p_mbuf(n) : stage_stride(n, 4), 16);
}
// the same in the streaming variant's ring (slots widened to a row buffer):
// measured slower at R = 1 for n = 14 / 16 (0.69 -> 0.51, 0.54 -> 0.50 of
// HBM; profiles/r01_f32p_ring_inplace.jsonl), so off
#ifndef JM_F32P_RING_INPLACE
#define JM_F32P_RING_INPLACE 0
#endif
JM_HD constexpr bool f32p_ring_inplace(int n) { return JM_F32P_RING_INPLACE && (n * n * 4) % 16 == 0; }

// Double-buffered (cp.async prefetch) staging.  Measured on B200 (r01 sweep):
// it lifts DMMA n=16 at repeat 1 from 0.87 to 0.94 of HBM, but the doubled
// stage area costs residency and the compute-bound repeat-100 configurations
// lose 1-25 % (FP32 row panels most), so those kinds run the single-buffered
// stage (their low-repeat variant is the bulk-copy ring instead).  The
// register-heavy thread-per-matrix sizes (f64 n = 5..7, f32 n = 8: 4-5
// CTAs per SM) do take it: +2-3 % at R = 100, +10-46 % at R <= 16
// (profiles/r01_tpm_stream_sweep.jsonl, r01_tpm_stream_hi.jsonl).
JM_HD constexpr bool prefetch_for(int n, int dtype) {
  return dtype == 1 ? (n >= 5 && n <= 7) : (n >= 8 && n <= JM_F32_TPM_MAX);
}

// ---- FP32 on the tensor cores, error-compensated TF32 (r02 late, run_f32tc) ----
// n a multiple of 16: a warp per matrix, P = M + M.M as m16n8k8 TF32 mma.sync
// tiles with each operand split x = hi + lo (hi = tf32(x), lo = tf32(x - hi))
// and the three products lo.hi + hi.lo + hi.hi accumulated in FP32 (the
// dropped lo.lo term is ~2^-22 relative).  The accumulator fragment of n-tile
// KS IS the A fragment of k-step KS under the k permutation (t, t+4) ->
// (2t, 2t+1), so only B (rows of M) goes through shared memory.
// JM_F32TC=1: the resident FP32 kernel of n = 16..JM_F32TC_MAXN (n % 16 == 0).
#ifndef JM_F32TC
#define JM_F32TC 1
#endif
#ifndef JM_F32TC_MAXN
#define JM_F32TC_MAXN 64
#endif
#ifndef JM_F32TC_16
#define JM_F32TC_16 0   // 1: n = 16 too (measurement hook)
#endif
// m-tiles (16 rows) per warp: the warps of a matrix split its rows (WPM =
// (n / 16) / MTW warps per matrix, a named barrier per matrix); each warp
// keeps its m-tiles' accumulators and A splits in registers
#ifndef JM_F32TC_MTW
#define JM_F32TC_MTW 0    // > 0: one value for every size
#endif
// n = 32, 40, 48, 56, 64 (profiles/r02_f32tc.md, fraction of the FP32 pipe
// at R = 100, with the non-finite check, FFMA2 tiles in brackets: 0.91 (0.77),
// 0.82 (0.66), 0.97 (0.76), 0.84 (0.66), 0.94 (0.78)); n = 16 (two accumulator
// fragments per warp: 0.69 against 0.72) and n = 24 (a half-padding m-tile:
// 0.67 against 0.73) stay on the FFMA2 tiles
#ifndef JM_F32TC_ALL
#define JM_F32TC_ALL 0   // 1: every multiple of 8 in 24..JM_F32TC_MAXN (measurement hook)
#endif
// n >= JM_F32TC_ODD that are not multiples of 8 take it too, zero-padded to
// 8*ceil(n/8) (profiles/r02_f32tc.md, R = 100: 38 0.60 -> 0.69, 41 0.55 ->
// 0.59, 44 0.65 -> 0.74, 47 0.73 -> 0.90, 50 0.56 -> 0.60, 53 0.59 -> 0.69,
// 57 0.59 -> 0.65, 60 0.65 -> 0.78, 63 0.73 -> 0.88; n = 35, padded to 40,
// loses: 0.67 -> 0.55).  0: off.
#ifndef JM_F32TC_ODD
#define JM_F32TC_ODD 37
#endif
JM_HD constexpr bool f32tc_use(int n) {
  return JM_F32TC && n <= JM_F32TC_MAXN &&
         ((n % 8 == 0 && n >= 32) || (n == 16 && JM_F32TC_16) || (JM_F32TC_ALL && n % 8 == 0 && n >= 24) ||
          (JM_F32TC_ODD > 0 && n % 8 != 0 && n >= JM_F32TC_ODD));
}
// (n a multiple of 8 but not of 16: the last m-tile is half padding rows,
// which never reach a real row: A row m only feeds P row m, and B reads rows k < n)
JM_HD constexpr int f32tc_mt(int n) { return ((n + 7) / 8 * 8 + 15) / 16; }                                  // m-tiles of a matrix
JM_HD constexpr int f32tc_mtw(int n) {
  return (JM_F32TC_MTW > 0 && f32tc_mt(n) % JM_F32TC_MTW == 0) ? JM_F32TC_MTW
         : n <= 48 ? f32tc_mt(n) : f32tc_mt(n) % 2 == 0 ? 2 : 1;   // one warp per matrix up to n = 48 (48: 0.97 vs 0.66 for three
                                        // warps, 40: 0.82 vs 0.54), two above (64: 0.94 vs 0.89 for four)
}
JM_HD constexpr int f32tc_wpm(int n) { return f32tc_mt(n) / f32tc_mtw(n); }                  // warps per matrix
JM_HD constexpr int f32tc_mpc(int n) { return f32tc_wpm(n) >= 4 ? 1 : 4 / f32tc_wpm(n); }   // matrices per CTA
JM_HD constexpr int f32tc_wpc(int n) { return f32tc_wpm(n) * f32tc_mpc(n); }
JM_HD constexpr int f32tc_ld(int n) { return (n + 7) / 8 * 8 + 4; }   // publish row stride (floats): B loads conflict free
JM_HD constexpr int f32tc_wbytes(int n) { return 16 * f32tc_mt(n) * f32tc_ld(n) * 4; }

JM_HD constexpr Plan plan_specialized(int n, int dtype) {
  const int es = dtype == 1 ? 8 : 4;
  const Tile t = tile_for(n, dtype);
  const int nst = prefetch_for(n, dtype) ? 2 : 1;   // stage buffers
  if (t == Tile::TPM) {
    return Plan{(int)t, TPM_THREADS, TPM_THREADS, nst * stage_bytes(TPM_THREADS, n, es), 1};
  }
  if (t == Tile::Reg)   // FP64 register tiles: the stage area IS the per-matrix region
    return Plan{(int)t, 32 * f32t_wpc(n, 1), f32t_mpc(n, 1), f32t_mpc(n, 1) * f32t_region(n, 1), f32t_wpm(n, 1)};
  if (t == Tile::Tpms) {
    return Plan{(int)t, TPM_THREADS, TPM_THREADS, stage_bytes(TPM_THREADS, n, es), 1};
  }
  if (t == Tile::Dmma) {
    const int w = dmma_w(n);
    if (w == 1)
      return Plan{(int)t, 32 * DMMA_WPC, DMMA_WPC,
                  nst * stage_bytes(DMMA_WPC, n, es) + DMMA_WPC * dmma_scr(n), 1};
    return Plan{(int)t, 32 * w, 1, nst * stage_bytes(1, n, es) + 2 * dmma_scr(n), w};
  }
  if (f32p_use(n)) {
    const int mpc = F32P_WPC * f32p_mpw(n);
    if (f32p_inplace(n)) return Plan{(int)Tile::F32Rows, 32 * F32P_WPC, mpc, nst * rup(mpc * f32p_slot(n), 16) + mpc * f32p_mbuf(n), 1};
    return Plan{(int)Tile::F32Rows, 32 * F32P_WPC, mpc, nst * stage_bytes(mpc, n, es) + mpc * f32p_pstr(n), 1};
  }
  if (dtype == 0 && f32tc_use(n))
    return Plan{(int)Tile::F32Tc, 32 * f32tc_wpc(n), f32tc_mpc(n), stage_bytes(f32tc_mpc(n), n, es) + f32tc_mpc(n) * f32tc_wbytes(n),
                f32tc_wpm(n)};
  // F32 tiles: the stage area IS the per-matrix region (stride f32t_region)
  return Plan{(int)t, 32 * f32t_wpc(n), f32t_mpc(n), f32t_mpc(n) * f32t_region(n), f32t_wpm(n)};
}

// Which entry point the specialization uses: k_update (maxThreads only) or
// k_update_mb1 (maxThreads, minBlocks = 1) — the CTA-per-matrix DMMA kinds.
JM_HD constexpr bool use_mb1(int n, int dtype, bool strm = false) {
  return tile_for(n, dtype) == Tile::Dmma && dmma_w(n, strm) > 1;
}
// ... or k_update[_stream]_rc (a register cap, __maxnreg__): the F32T tiles
JM_HD constexpr bool use_rc(int n, int dtype, bool strm = false) {
  return (dtype == 0 && tile_for(n, dtype) == Tile::F32 && (strm ? f32t_stream_use(n) : f32t_use(n) && !f32tc_use(n))) ||
         tile_for(n, dtype) == Tile::Reg;
}

// ---- streaming variant (low repeat: the HBM-bound side of the roofline) ----
// At R(n+1) below the ridge (R(n+1) < 46 for both dtypes) the
// update is bound by moving each matrix in and out once, and the resident
// kinds above, which load -> compute -> store each chunk in turn, leave HBM
// idle while they compute.  The streaming variant runs the SAME tiling kinds
// (same compute code, same round of MPC matrices) behind a bulk-copy ring
// (jm::Ring): chunks of K rounds, JM_RING_S stages deep, ~JM_RING_CHUNK bytes
// each.  The host picks it per call from the repeat count (stream_rn); it is a
// second cache key of the same (N, dtype, addend).
// TPM (thread per matrix) keeps its resident kernel: its per-thread reads need
// the odd-16-B staging stride, and it already streams at 0.89-0.99 of HBM.
#ifndef JM_RING_S
#define JM_RING_S 2
#endif
#ifndef JM_RING_NOWAIT_UNSAFE
#define JM_RING_NOWAIT_UNSAFE 0   // timing experiment only (wrong results): skip the store-read wait before a refill
#endif
#ifndef JM_RING_CHUNK
#define JM_RING_CHUNK 8192
#endif
// (for Tile::TPM the streaming variant is the same thread-per-matrix kernel
// with the double-buffered cp.async stage: its per-thread reads need the
// odd-16-B staging stride, which a bulk copy per matrix would make 1-D copies
// of 32..512 B)
JM_HD constexpr bool stream_ok(int n, int dtype) {
  return tile_for(n, dtype) == Tile::Dmma || tile_for(n, dtype) == Tile::F32 || tile_for(n, dtype) == Tile::Reg ||
         tile_for(n, dtype) == Tile::Tpms ||
         tile_for(n, dtype) == Tile::TPM;
}
// The host's switch: stream iff repeat * (n + 1) < stream_rn(n, dtype).
// Placed from the measured crossovers (profiles/r01_stream_sweep*.jsonl and
// r01_stream_xover.jsonl, one B200): the ring costs shared memory, hence
// residency, and above n = 32 the streaming variant also keeps the narrower
// CTA mapping, so it wins while the load/store half of the roofline still
// matters and loses once the update is compute-bound.  f64: n = 9..32 gains up
// to R(n+1) ~ 600 (n = 32: 1.96x at R = 1, 1.18x at R = 8); n = 33 / 34 (the
// resident kernel has the thin border there) only at R <= 2; 35..40 to ~300;
// 41..48 to ~250; 49..56 to ~600; 57..64 to ~400; n = 8 loses 8 % at R = 1
// (16 copies of 512 B per chunk) and stays resident; n = 9, 10 see JM_TPMS_RN.
// f32: row panels (n = 15, 16) gain to ~64; the tiles (n >= 17) stream
// through their prefetching stage below JM_F32T_RN; the staged-product sizes
// (12..14) and the thread-per-matrix sizes have their own rules below.
// n = 9, 10: the DMMA ring streams better only at R = 1 (0.68 vs 0.56 of HBM);
// from R = 2 the staged-product kind wins (R = 100: 0.65 / 0.68 of the FP64
// pipe vs 0.22 / 0.24 for the padded DMMA tile; profiles/r01_tpms_n9_10.jsonl)
#ifndef JM_TPMS_RN
#define JM_TPMS_RN 20
#endif
JM_HD constexpr int stream_rn_f64(int n) {
  return (n >= 9 && n <= JM_F64_TPMS_MAX) ? JM_TPMS_RN : n <= 8 ? 0 : n <= 32 ? 600 : n <= 34 ? 100 : n <= 40 ? 300 : n <= 48 ? 250 : n <= 56 ? 600 : 400;
}
// ... and not below stream_lo(n, dtype): f64 n = 16 at R = 1, whose resident
// kernel (16 KB, 48 registers: 40 warps per SM) streams at 0.95 of HBM once
// its accumulator loads are conflict free, against 0.88 through the ring
// (profiles/r01_ring_lowr_sweep.jsonl; from R = 2 the ring wins, 0.91 vs 0.80)
JM_HD constexpr int stream_lo(int n, int dtype) {
  return (dtype == 1 && n == 16) ? 18 : (dtype == 0 && n == 3) ? 32 : 0;
}
// Thread per matrix (profiles/r01_tpm_stream_sweep.jsonl): the staged
// variant wins where registers limit the resident kernel to few CTAs — f64
// n = 5..7 (1.14-1.46x at R = 1..8; n = 6 R = 1: 0.66 -> 0.94 of HBM) and
// f32 n = 8..11 — at every R, so those sizes' resident kernel prefetches
// itself (prefetch_for); it loses up to 23 % on the small, light sizes (f64
// n = 2: 0.96 -> 0.74 of HBM).  So the TPM streaming key is normally not picked.
// One exception: f32 n = 3 gains from the staged variant once R >= 8
// (1.13x at R = 8, 1.05x at R = 100) and loses below (0.89x at R = 1), so it
// streams above the lower bound stream_lo (r01_all_n_sweep.jsonl,
// r01_tpm_stream_sweep.jsonl).
// FP64 register tiles: the DMMA ring wins below this R(n+1) (R = 1: 0.69-0.90
// of HBM against 0.31-0.47 for the register tiles; crossovers measured at
// R = 1..16, profiles/r02_f64t_xover.jsonl: n = 11, 12 ~ 100-140, 18 ~ 150,
// 19, 20 ~ 300)
#ifndef JM_F64T_RN
#define JM_F64T_RN 0     // > 0: one switch point for every register-tile size
#endif
JM_HD constexpr int f64t_rn(int n) { return JM_F64T_RN > 0 ? JM_F64T_RN : n <= 12 ? 120 : n <= 18 ? 160 : 330; }
// FP32 register tiles: the streaming kernel (ring / prefetching stage, with
// its own tile shapes, F32TS_TABLE) while R <= F32T_STREAM_MAXR[n]: measured
// stream vs resident at R = 2..12, 24 and 100 (profiles/r02_f32_stream_xover_v3.jsonl,
// r02_f32_stream_xover_r24_r100.jsonl).  With its two-warp CTAs and shapes the
// streaming kernel is the faster one even at R = 100 for n = 27, 29, 31, 32,
// 34, 36, 38, 39, 41, 45, 46, 52, 54, 55, 58..60 (e.g. n = 52 0.54 -> 0.56,
// 60 0.61 -> 0.65 of the pipe), so those sizes always stream (1 << 20).
// JM_F32T_RN > 0: one switch point R(n+1) < JM_F32T_RN for every tile size.
#ifndef JM_F32T_RN
#define JM_F32T_RN 0
#endif
constexpr int F32T_STREAM_MAXR[65] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 24, 6, 10, 8, 50, 50, 12, 8, 10, 8, 50, 1048576, 12, 1048576, 50, 1048576, 2, 8, 1048576, 24, 1048576, 4, 4, 4, 1, 4, 4, 4, 4, 4, 4, 4, 1, 4, 4, 4, 4, 4, 4, 4, 1, 8, 8, 8, 8, 8, 8, 8, 3};
// (n = 32, 40, 48, 56, 64: the resident kernel is the tensor-core kind,
// run_f32tc; measured crossovers (profiles/r02_f32tc_xover*.jsonl): n = 32 and
// 64 tie the streaming tiles at R = 3, n = 40, 48, 56 win from R = 2 (0.58 vs
// 0.49, 0.64 vs 0.62, 0.66 vs 0.60 of the pipe) — so 32 streams at R <= 2,
// 64 at R <= 3, 40 / 48 / 56 at R = 1 only; the zero-padded sizes 37..63
// stream to R = 4 (<= 56) / 8 (57..63): at R = 8 the padded kernel wins
// except n = 57 (0.51 vs 0.55) and 63 (a tie))
JM_HD constexpr int f32t_rn(int n) {
  return JM_F32T_RN > 0 ? JM_F32T_RN
         : F32T_STREAM_MAXR[n] >= (1 << 20) ? (1 << 30)
         : F32T_STREAM_MAXR[n] > 0 ? F32T_STREAM_MAXR[n] * (n + 1) + 1 : 9 * (n + 1);
}
JM_HD constexpr int stream_rn_tpm(int n, int dtype) { return (dtype == 0 && n == 3) ? (1 << 30) : 0; }
JM_HD constexpr int stream_rn(int n, int dtype) {
  return !stream_ok(n, dtype)               ? 0
         : tile_for(n, dtype) == Tile::TPM ? stream_rn_tpm(n, dtype)
         : tile_for(n, dtype) == Tile::Reg ? f64t_rn(n)
         : (dtype == 0 && tile_for(n, dtype) == Tile::Tpms) ? (n == 12 ? 0 : 20)   // R = 1: row-panel ring
         : dtype == 1        ? stream_rn_f64(n)
         : (f32p_use(n) && !f32t_stream_use(n)) ? 64
                             : f32t_rn(n);
}
// rounds per chunk: >= JM_RING_CHUNK bytes and a chunk a multiple of 16 B
JM_HD constexpr int ring_k(int rb) {
  return rup(cdiv(JM_RING_CHUNK, rb), (rb % 16 == 0) ? 1 : (rb % 8 == 0) ? 2 : 4);
}
// matrix stride in a ring stage: the odd-16-B stage stride when a matrix is a
// multiple of 16 B (one bulk copy per matrix), else packed (one per chunk)
// (slot: a larger per-matrix slot a kind wants to work in, see dmma_slot)
JM_HD constexpr int ring_sbm(int n, int es, int slot = 0) {
  return (n * n * es) % 16 == 0 ? (slot > stage_stride(n, es) ? slot : stage_stride(n, es)) : n * n * es;
}
// r02, shifted per-matrix copies: an FP64 matrix of odd n is 8 B short of a
// whole number of 16-B pieces, so one matrix per round (the CTA-DMMA ring)
// needed chunks of two matrices (K = 2).  Instead each matrix sits at byte
// (global offset mod 16) of a slot of n*n*8 + 8 bytes: its 16-B-aligned body is
// one bulk copy, the 8 bytes outside it one cp.async tied to the same mbarrier
// (cp.async.mbarrier.arrive) — chunks of ONE matrix, half the ring.
// JM_RING_SHIFT=0: off.
// Streaming CTA-DMMA kernels (W > 1, publish buffer not in the ring slot):
// one publish buffer + one more CTA barrier per update instead of two
// alternating buffers (run_dmma ONE), where two buffers would leave one CTA
// per SM (> JM_DMMA_1BUF_MAXB): odd n = 57..63 then fit two.  Measured
// (profiles/r02_ab_dmma_stream_1buf.md, FP64 pipe at R = 1): 57 0.41 -> 0.55,
// 59 0.45 -> 0.59, 61 0.47 -> 0.63, 63 0.51 -> 0.68; where it does not change
// the CTAs per SM the extra barrier costs up to 0.05 (n = 56), so only there.
// JM_DMMA_STREAM_1BUF=0: two buffers everywhere.
#ifndef JM_DMMA_STREAM_1BUF
#define JM_DMMA_STREAM_1BUF 1
#endif
#ifndef JM_DMMA_1BUF_MAXB
#define JM_DMMA_1BUF_MAXB (113 * 1024)
#endif
#ifndef JM_RING_SHIFT
#define JM_RING_SHIFT 1
#endif
JM_HD constexpr bool ring_shift(int n, int es, int rm) {
  return JM_RING_SHIFT && es == 8 && rm == 1 && (n * n * es) % 16 == 8;
}
JM_HD constexpr int ring_kr(int n, int es, int rm) {   // rounds per chunk
  return ring_shift(n, es, rm) ? cdiv(JM_RING_CHUNK, n * n * es) : ring_k(rm * n * n * es);
}
JM_HD constexpr int ring_sbmr(int n, int es, int rm, int slot = 0) {   // matrix slot stride
  return ring_shift(n, es, rm) ? (slot > n * n * es + 8 ? slot : n * n * es + 8) : ring_sbm(n, es, slot);
}
JM_HD constexpr int ring_bytes(int n, int es, int rm, int slot = 0) {
  return JM_RING_S * ring_kr(n, es, rm) * rm * ring_sbmr(n, es, rm, slot) + rup(8 * JM_RING_S, 16);
}
// DMMA in the streaming variant: when the swizzled publish buffer fits in the
// matrix's ring slot (n a multiple of 16), the slot is reused as that buffer
// (W == 1) or as the first of the two (W > 1) once M sits in the accumulators:
// n = 32 then holds 3 CTAs per SM instead of 2, n = 48 / 64 two instead of one
// For other even n the slot can be widened to the publish buffer's size
// (dmma_slot), one ring slot per matrix instead of a slot plus a separate
// buffer.  Measured (profiles/r01_dmma_ring_slot.jsonl, R = 1): it pays where
// it lifts the CTAs per SM — n = 26..30 (2 -> 3 CTAs: 0.65 -> 0.76 of HBM at
// n = 28) and 58..62 (1 -> 2: 0.37 -> 0.45 at n = 62) — and is noise or a
// loss elsewhere (n = 56: 0.54 -> 0.49), so it is applied there only
// (JM_DMMA_RING_SLOT=0: never, =2: every even n).
#ifndef JM_DMMA_RING_SLOT
#define JM_DMMA_RING_SLOT 1
#endif
JM_HD constexpr int dmma_slot(int n) {
  return (n % 2 == 0 && dmma_scr(n) > ring_sbm(n, 8) &&
          (JM_DMMA_RING_SLOT == 2 || (JM_DMMA_RING_SLOT == 1 && ((n >= 26 && n <= 30) || n >= 58))))
             ? dmma_scr(n) : 0;
}
JM_HD constexpr bool dmma_inplace(int n) { return dmma_scr(n) <= ring_sbm(n, 8, dmma_slot(n)); }
// FP32 tiles' low-repeat variant: the bulk-copy ring with slots widened to the
// work region when a matrix is a multiple of 16 B (even n: one bulk copy per
// matrix); odd n keep the double-buffered cp.async stage.  JM_F32T_RING=0: off.
#ifndef JM_F32T_RING
#define JM_F32T_RING 1
#endif
// n % 4 == 0: rotated 16-B one-time reads / write-backs of the packed matrix
// (run_f32t PVEC), in the low-repeat (streaming) kernel, where the one-time
// accesses are a large share of the shared-memory traffic (at R = 100 they are
// noise).  First measured with the resident tile shapes (profiles/r02_ab_pvec.md,
// R = 1: 20 0.67 -> 0.75, 32 0.65 -> 0.76, but 24 0.71 -> 0.67), then the
// streaming shapes were searched with the one-time accesses in the layout model
// (tools/f32_layout.py init_wavefronts) and PVEC on.  JM_F32T_PVEC=0: off.
#ifndef JM_F32T_PVEC
#define JM_F32T_PVEC 1
#endif
JM_HD constexpr bool f32t_pvec(int n, bool strm) {   // (resident n = 60: +0.03 of the pipe at R = 100)
  return JM_F32T_PVEC && (strm || n == 60) && (n % 4) == 0;
}
#ifndef JM_F32T_RING_ROWS
#define JM_F32T_RING_ROWS 0   // 1: row-pitched copies straight into the work layout (run_f32t RROWS); measured 2-5x slower at R = 1 (one 80-256 B bulk copy per row, profiles/r02_ab_f32_ring_rows.md)
#endif
#ifndef JM_F32T_RING_MAXB
#define JM_F32T_RING_MAXB (113 * 1024)   // ... while two CTAs still fit on an SM
#endif
// JM_F32T_SEP_ALL: every n takes the packed ring with separate work regions
// (f32t_ring_sep), not the in-place ring.  Measured at R = 1..2 for n = 17..64
// (profiles/r02_ab_f32_stream_sep.md): the chunk-wise copy into a separate work
// region removes the conflicted element reads of the packed matrix, but the
// extra region costs occupancy (n = 20 0.64 -> 0.47, 40 0.50 -> 0.41 of HBM;
// n = 32 / 48 +2-4 %), and the element-wise copy of rows that are not whole
// 16-B chunks is slower still (n = 18 0.61 -> 0.23) — off
#ifndef JM_F32T_SEP_ALL
#define JM_F32T_SEP_ALL 0
#endif
JM_HD constexpr bool f32t_ring(int n) {
  return JM_F32T_RING && !JM_F32T_SEP_ALL && (n * n * 4) % 16 == 0 &&
         ring_bytes(n, 4, f32t_mpc(n, 2), f32t_region(n, 2)) <= JM_F32T_RING_MAXB;
}
// odd n: the ring of packed chunk copies (a matrix is not a multiple of 16 B,
// so it cannot be its own copy into a slot) beside a separate work region per
// matrix of the round, while that still fits twice on an SM.  Measured slower
// than the prefetching stage (n = 25 0.37 -> 0.26, 27 0.46 -> 0.23 of HBM at
// R = 1; profiles/r02_ab_f32_stream_sep.md) — off
#ifndef JM_F32T_RING_SEP
#define JM_F32T_RING_SEP 0
#endif
JM_HD constexpr bool f32t_ring_sep(int n) {
  return JM_F32T_RING_SEP && (JM_F32T_SEP_ALL || (n * n * 4) % 16 != 0) &&
         ring_bytes(n, 4, f32t_mpc(n, 2)) + f32t_mpc(n, 2) * f32t_region(n, 2) <= JM_F32T_RING_MAXB;
}
// odd n without the ring (the low-repeat kernel is the prefetching cp.async
// stage): each matrix is staged at byte (its global offset & 15) of its
// region, so it moves by 16-B copies instead of one 4-B copy per element each
// way (run_f32t PSH, Stager SHIFT); needs 12 spare bytes in the region.
// Measured at R = 1 (profiles/r02_ab_f32_pshift.md, fraction of HBM): a gain
// only where a CTA holds one or two matrices, n >= 55 (55 0.33 -> 0.37, 59
// 0.41 -> 0.43, 63 0.42 -> 0.48); for n = 17..23 the per-matrix head / tail
// work costs more than the element copies it replaces (17 0.45 -> 0.37), and
// 25..53 are within noise.  JM_F32T_PSHIFT=0: off; JM_F32T_PSHIFT_MIN: the
// smallest n that takes it.
#ifndef JM_F32T_PSHIFT
#define JM_F32T_PSHIFT 1
#endif
#ifndef JM_F32T_PSHIFT_MIN
#define JM_F32T_PSHIFT_MIN 55
#endif
JM_HD constexpr bool f32t_pshift(int n) {
  return JM_F32T_PSHIFT && n >= JM_F32T_PSHIFT_MIN && (n * n * 4) % 16 != 0 && n * n * 4 + 12 <= f32t_region(n, 2);
}
// matrices per round of each kind (the resident plan's chunk)
JM_HD constexpr int round_mpc(int n, int dtype) {
  return (tile_for(n, dtype) == Tile::Dmma ||
          (dtype == 1 && (tile_for(n, dtype) == Tile::Tpms || tile_for(n, dtype) == Tile::Reg)))
             ? (dmma_w(n, true) == 1 ? DMMA_WPC : 1)
         : (f32p_use(n) && !f32t_stream_use(n)) ? F32P_WPC * f32p_mpw(n)
                                         : f32t_mpc(n, 2);
}
JM_HD constexpr bool dmma_stream_1buf(int n) {
  return JM_DMMA_STREAM_1BUF && dmma_w(n, true) > 1 && !dmma_inplace(n) &&
         ring_bytes(n, 8, 1, dmma_slot(n)) + 2 * dmma_scr(n) > JM_DMMA_1BUF_MAXB;
}
// Plan of the streaming variant: mpc = matrices per ring chunk (the host sizes
// the grid by it); smem = the ring + the kind's own work areas.
JM_HD constexpr Plan plan_stream(int n, int dtype) {
  const int es = dtype == 1 ? 8 : 4;
  const int rm = round_mpc(n, dtype), chm = ring_kr(n, es, rm) * rm;
  if (!stream_ok(n, dtype)) return plan_specialized(n, dtype);
  if (tile_for(n, dtype) == Tile::TPM)
    return Plan{(int)Tile::TPM, TPM_THREADS, TPM_THREADS, 2 * stage_bytes(TPM_THREADS, n, es), 1};
  if (tile_for(n, dtype) == Tile::Dmma ||
      (dtype == 1 && (tile_for(n, dtype) == Tile::Tpms || tile_for(n, dtype) == Tile::Reg))) {   // (Tpms, Reg: DMMA ring)
    const int w = dmma_w(n, true);
    const int own = dmma_inplace(n) ? (w == 1 ? 0 : 1) : (w == 1 ? DMMA_WPC : (dmma_stream_1buf(n) ? 1 : 2));   // scratch buffers
    return Plan{(int)Tile::Dmma, 32 * (w == 1 ? DMMA_WPC : w), chm, ring_bytes(n, es, rm, dmma_slot(n)) + own * dmma_scr(n), w};
  }
  if (f32p_use(n) && !f32t_stream_use(n))
    return f32p_ring_inplace(n)
               ? Plan{(int)Tile::F32Rows, 32 * F32P_WPC, chm, ring_bytes(n, es, rm, f32p_slot(n)) + rm * f32p_mbuf(n), 1}
               : Plan{(int)Tile::F32Rows, 32 * F32P_WPC, chm, ring_bytes(n, es, rm) + rm * f32p_pstr(n), 1};
  // F32T, even n: the bulk-copy ring, each matrix's slot widened to its work
  // region (the staged matrix is read into the accumulators, then the slot is
  // the work area; the result goes back packed and leaves by a bulk store)
  if (f32t_ring(n))
    return Plan{(int)Tile::F32, 32 * f32t_wpc(n, 2), chm, ring_bytes(n, es, rm, f32t_region(n, 2)), f32t_wpm(n, 2)};
  if (f32t_ring_sep(n))
    return Plan{(int)Tile::F32, 32 * f32t_wpc(n, 2), chm, ring_bytes(n, es, rm) + rm * f32t_region(n, 2),
                f32t_wpm(n, 2)};
  // F32T, odd n: the resident layout with the double-buffered cp.async stage
  // (the next chunk streams in while this one is updated)
  return Plan{(int)Tile::F32, 32 * f32t_wpc(n, 2), f32t_mpc(n, 2), 2 * rup(f32t_mpc(n, 2) * f32t_region(n, 2), 16),
              f32t_wpm(n, 2)};
}

// Note: k_update passes only maxThreads to __launch_bounds__.  Registers are
// granted per SMSP (16384 each), so a minBlocks cap only bites in steps of
// warps-per-SMSP (2 -> 255, 3 -> 168 regs); 168 makes the FP32 row panels
// spill, and an explicit minBlocks = 1 changes ptxas' heuristics (r01: TPM
// f32 n=2 went 32 -> 45 registers and lost 18 % of HBM throughput).

// ---- latency path (tiny batches; BASELINE.json configs[0] "C1") ----
// A thread-per-matrix kernel runs each matrix's N^2 (N+1) FMAs per update on
// ONE thread; with few matrices the GPU idles and one update costs ~200 SM
// clocks (r01 C1: 1 x 4x4 x 1000 updates in 109 us, slower than a CPU core).
// k_update_lat gives each matrix a warp, lane i*N+j owning M[i][j], and forms
// P[i][j] with N shuffled pairs: the per-update critical path is one N-long
// FMA chain.  For N*N <= 32; chosen when the batch is at most LAT_BATCH_PER_SM
// matrices per SM (each matrix then has its own warp) or by JM_FLAG_LATENCY.
constexpr int LAT_THREADS = 128;                   // 4 matrices (warps) per CTA
constexpr int LAT_BATCH_PER_SM = 4;
JM_HD constexpr bool lat_ok(int n) { return n * n <= 32; }
JM_HD constexpr Plan plan_lat(int n, int dtype) {
  return Plan{(int)Tile::Lat, LAT_THREADS, LAT_THREADS / 32, 0, (n + dtype) > 0 ? 1 : 1};
}

// ---- AoT specializations (nvcc-compiled at build time; Fig. 3's sizes) ----
JM_HD constexpr bool aot_spec_available(int n, int dtype) {
  return dtype == 1 && (n == 3 || n == 7 || n == 16);
}

// ---- batched multiply-accumulate (Listing 8) ----
constexpr int MM_THREADS = 256;
JM_HD constexpr int mm_mpc(int n) { return (n * n >= MM_THREADS) ? 1 : MM_THREADS / (n * n); }
// Specialized multiply-accumulate: a bulk-copy (TMA, cp.async.bulk) ring of
// MM_STAGES chunk buffers, each holding MPC packed matrices of A, B and C.  A
// chunk's byte count must be a multiple of 16, so MPC is a multiple of
// 16 / gcd(MB, 16); about MM_CHUNK_BYTES per operand per chunk.
constexpr int MM_CHUNK_BYTES = 8192;
constexpr int MM_STAGES_MAX = 4;
constexpr int MM_SMEM_BUDGET = 200 * 1024;
constexpr int MM_BAR_BYTES = 64;  // MM_STAGES_MAX mbarriers, padded
JM_HD constexpr int mm_align_mult(int mb) { return (mb % 16 == 0) ? 1 : (mb % 8 == 0) ? 2 : 4; }
JM_HD constexpr int mm_bulk_mpc(int n, int es) {
  const int mb = n * n * es, m = mm_align_mult(mb);
  const int k = (MM_CHUNK_BYTES / mb) / m * m;
  return k > 0 ? k : m;
}
JM_HD constexpr int mm_bulk_stages(int n, int es) {
  const int s = MM_SMEM_BUDGET / (3 * mm_bulk_mpc(n, es) * n * n * es);
  return s > MM_STAGES_MAX ? MM_STAGES_MAX : s;
}
// sizes whose chunk ring does not fit twice (large odd n) keep the staged path
JM_HD constexpr bool mm_bulk(int n, int es) { return mm_bulk_stages(n, es) >= 2; }
// Small batches (fewer full chunks than SMs) are latency-bound: the ring would
// leave most SMs idle, so the kernel computes straight from global memory over
// the whole grid instead and is launched without the ring's shared memory.
constexpr int MM_DIRECT_CHUNKS = 148;
JM_HD constexpr bool mm_direct(long long batch, int n, int es) {
  return !mm_bulk(n, es) ? false : batch < (long long)MM_DIRECT_CHUNKS * mm_bulk_mpc(n, es);
}
constexpr int MM_DIRECT_GRID = 148 * 8;  // 2048 threads per SM
JM_HD constexpr Plan plan_matmul(int n, int dtype) {
  const int es = dtype == 1 ? 8 : 4;
  if (mm_bulk(n, es)) {
    const int mpc = mm_bulk_mpc(n, es);
    return Plan{(int)Tile::Generic, MM_THREADS, mpc, mm_bulk_stages(n, es) * 3 * mpc * n * n * es + MM_BAR_BYTES, 1};
  }
  return Plan{(int)Tile::Generic, MM_THREADS, mm_mpc(n), 2 * stage_bytes(mm_mpc(n), n, es), 1};
}
// the AoT generic (runtime n) kernel: A and B staged per chunk, C streamed
JM_HD constexpr Plan plan_matmul_generic(int n, int dtype) {
  return Plan{(int)Tile::Generic, MM_THREADS, mm_mpc(n), 2 * stage_bytes(mm_mpc(n), n, dtype == 1 ? 8 : 4), 1};
}

// ---- Laghos 2D mass operator (Listing 12) ----
// one thread per element, MASS_THREADS elements per CTA chunk
constexpr int MASS_MAX = 8;                        // 1 <= D, Q <= 8 (Fig. 7: d,q in {2,4,8})
constexpr int MASS_THREADS = 64;
#ifndef JM_MASS_PF
#define JM_MASS_PF 1                 // thread-per-element kernel: double-buffered cp.async staging
#endif
// ... except the tiniest elements, where the doubled stage area costs more
// residency than the overlap gains ((1, 1) 0.53 -> 0.49, (2, 1) 0.71 -> 0.64,
// (2, 2) 0.70 -> 0.61 of HBM; every other pair gains, up to 0.41 -> 0.99:
// profiles/r02_mass_pf_ab.jsonl)
JM_HD constexpr bool mass_pf(int d, int q) { return JM_MASS_PF && !((d == 1 && q == 1) || (d == 2 && q <= 2)); }
// r02: the DMMA kernel (a warp per element, the four contractions on the FP64
// tensor cores, D and Q padded to 8; jm_mass.cuh mass_dmma_body) for the
// (D, Q) where it measured faster than the thread-per-element kernel, whose
// D*Q*(D+Q) FMAs per element each take a broadcast shared load of B (the DMMA
// kernel's cost per element is fixed: 8 DMMA).  All 64 pairs at 2^21
// elements, fraction of HBM (profiles/r02_mass_ab.md): against r01's
// single-buffered thread kernel D = 8 0.29-0.52 -> 0.93-1.05, D = 6, 7
// 0.27-0.60 -> 0.65-0.82; the thread kernel then got double-buffered cp.async
// staging (JM_MASS_PF: median 0.69 -> 0.87 of HBM over all pairs) and wins
// again below D*Q ~ 30-40: the table is from that comparison
// (r02_mass_table_ab.jsonl): D = 8 Q >= 2, D = 7 Q >= 4, D = 6 Q >= 6,
// D = 4, 5 Q = 8.  Row d of the table: bit q-1 set = DMMA.  MASS_DMMA_THREADS
// / 32 elements per CTA chunk.  JM_MASS_DMMA: 0 the table, 1 every pair, -1
// none (A/B builds)
#ifndef JM_MASS_DMMA
#define JM_MASS_DMMA 0
#endif
#ifndef JM_MASS_DMMA_PD
#define JM_MASS_DMMA_PD 4            // elements per warp in flight (cp.async slots per warp)
#endif
#ifndef JM_MASS_DMMA_MINB
#define JM_MASS_DMMA_MINB 4          // __launch_bounds__ min CTAs per SM (<= 64 registers; 4 CTAs also fill the shared memory at PD = 4)
#endif
constexpr int MASS_DMMA_THREADS = 256;
constexpr int MASS_DMMA_SLOT = 1536;   // one element's x, y, op fragments for 32 lanes (3 x 512 B)
JM_HD constexpr unsigned mass_dmma_row(int d) {   // (r02, against the double-buffered thread kernel)
  return d == 8 ? 0xfeu : d == 7 ? 0xf8u : d == 6 ? 0xe0u : d >= 4 ? 0x80u : 0u;
}
JM_HD constexpr bool mass_dmma(int d, int q) {
  return JM_MASS_DMMA > 0 || (JM_MASS_DMMA == 0 && ((mass_dmma_row(d) >> (q - 1)) & 1u));
}
JM_HD constexpr Plan plan_mass(int d, int q) {
  return mass_dmma(d, q)
             ? Plan{(int)Tile::Dmma, MASS_DMMA_THREADS, MASS_DMMA_THREADS / 32,
                    MASS_DMMA_THREADS / 32 * JM_MASS_DMMA_PD * MASS_DMMA_SLOT, 1}
             : Plan{(int)Tile::Generic, MASS_THREADS, MASS_THREADS,
                    (mass_pf(d, q) ? 2 : 1) * (2 * stage_bytes(MASS_THREADS, d, 8) + stage_bytes(MASS_THREADS, q, 8)) +
                        rup(q * d * 8, 16), 1};
}

// ---- GENERIC (runtime N; AoT) ----
constexpr int GENERIC_THREADS = 256;
JM_HD constexpr int generic_mpc(int n) { return (n * n >= GENERIC_THREADS) ? 1 : GENERIC_THREADS / (n * n); }
JM_HD constexpr Plan plan_generic(int n, int dtype) {
  // staging area + product buffer, both packed n*n per matrix
  return Plan{(int)Tile::Generic, GENERIC_THREADS, generic_mpc(n),
              2 * generic_mpc(n) * n * n * (dtype == 1 ? 8 : 4), 1};
}

}  // namespace jm
#endif  // JM_PLAN_H
