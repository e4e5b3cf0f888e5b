#!/usr/bin/env python3
"""Register-tile shape and shared-memory layout search for the FP32 tiles (run_f32t).

    python tools/f32_layout.py [--n 17..64] [--top 5] [--emit]

For each n it enumerates register tiles RA x CB (RG x CG threads per matrix),
row strides LDM, per-matrix region padding and column mappings, and scores
them with a cost model:

* shared-memory wavefronts of every LDS.128 / STS.128 a warp issues per update
  (A loads M[row][4kb..4kb+3], B loads row k, the publish of M), under the
  model measured on B200 by tools/microbench/lds_wavefronts.cu (ncu,
  profiles/r02_lds_wavefronts.md): each half-warp costs one wavefront when its
  two quarter-warps' addresses fall in disjoint 16-B bank slots with at most
  one address per slot (or all its lanes read one address), else the sum of
  the quarters' costs (a quarter costs its largest number of distinct
  addresses in one slot); the SM serves one wavefront per clock and two FFMA2
  warp-instructions per clock;
* padding (n^2 useful of NR x NC computed; k is exact), idle lanes;
* registers (accumulators + A block + two B rows + ~12) -> warps per SMSP,
  and shared memory per matrix -> warps per SM.

--emit prints the jm_plan.h table (f32t_table) of the best candidate per n.
"""
from __future__ import annotations

import argparse
from dataclasses import dataclass


def cdiv(a, b):
    return -(-a // b)


def rup(a, b):
    return cdiv(a, b) * b


def wavefronts(addrs: dict[int, int]) -> int:
    """addrs: lane -> byte address (active lanes only) of one 128-bit access."""
    tot = 0
    for h in (0, 1):
        lanes = [l for l in range(16 * h, 16 * h + 16) if l in addrs]
        if not lanes:
            continue
        if len({addrs[l] for l in lanes}) == 1:
            tot += 1
            continue
        qs = []
        for q in (0, 1):
            ql = [l for l in lanes if (l - 16 * h) // 8 == q]
            qs.append({addrs[l] for l in ql})

        def cost(aset):
            if not aset:
                return 0
            slots = {}
            for a in aset:
                slots.setdefault((a // 16) % 8, set()).add(a)
            return max(len(v) for v in slots.values())

        u = qs[0] | qs[1]
        if not (qs[0] & qs[1]) and cost(u) <= 1:
            tot += 1
        else:
            tot += cost(qs[0]) + cost(qs[1])
    return tot


@dataclass
class Cand:
    n: int
    ra: int
    cb: int
    rg: int
    cg: int
    ldm: int
    pad: int
    colblk: int
    trfast: int = 1       # 1: tr = t % RG (thread rows fastest), 0: tc = t % CG
    qmix: int = 0         # 1 (two matrices per warp): quarter-warps alternate matrices
    es: int = 4           # element size: 4 float (FFMA2 tiles), 8 double (DFMA tiles)
    wpc: int = 4

    @property
    def tpmat(self):
        return self.rg * self.cg

    @property
    def wpm(self):
        return cdiv(self.tpmat, 32) if self.tpmat > 32 else 1

    @property
    def mpw(self):
        return 1 if self.tpmat > 32 else 2 if self.qmix else 32 // self.tpmat

    @property
    def nr(self):
        return self.rg * self.ra

    @property
    def nc(self):
        return self.cg * self.cb

    @property
    def vec(self):           # elements per 16-B chunk
        return 16 // self.es

    @property
    def srows(self):
        return max(self.nr, rup(self.n, self.vec))

    @property
    def region(self):
        return rup(max(self.srows * self.ldm * self.es, self.n * self.n * self.es), 16) + 16 * self.pad

    @property
    def regs(self):
        return (self.es // 4) * (self.ra * self.cb + self.vec * self.ra + 2 * self.cb) + 14

    def row(self, i, tr):
        return i * self.rg + tr

    def lanes(self, warp):
        """(lane, mi, tr, tc) of the live lanes of warp `warp` of a CTA."""
        out = []
        for lane in range(32):
            if self.wpm == 1:
                if self.qmix:      # quarters q = lane / 8: matrix q % 2, threads (q / 2) * 8 + lane % 8
                    m, t = (lane // 8) % 2, (lane // 16) * 8 + lane % 8
                else:
                    m, t = lane // self.tpmat, lane % self.tpmat
                if m >= self.mpw or t >= self.tpmat:
                    continue
                mi = warp * self.mpw + m
            else:
                t = (warp % self.wpm) * 32 + lane
                if t >= self.tpmat:
                    continue
                mi = warp // self.wpm
            tr, tc = (t % self.rg, t // self.rg) if self.trfast else (t // self.cg, t % self.cg)
            out.append((lane, mi, tr, tc))
        return out

    def chunk(self, h, tc):
        nh = self.cb // self.vec
        return tc * nh + h if self.colblk else h * self.cg + tc

    def update_wavefronts(self, warp=0):
        """wavefronts of one update (per warp): A + B loads, publish."""
        L = self.lanes(warp)
        nh = self.cb // self.vec
        rowb = self.ldm * self.es
        wa = wb = ws = 0
        # (a k block / a k step shifts every lane's address by the same 16 B /
        # row stride, so one block / one step stands for all of them)
        for i in range(self.ra):
            wa += cdiv(self.n, self.vec) * wavefronts({l: mi * self.region + self.row(i, tr) * rowb
                                                       for l, mi, tr, tc in L})
            for h in range(nh):
                ws += wavefronts({l: mi * self.region + self.row(i, tr) * rowb + 16 * self.chunk(h, tc)
                                  for l, mi, tr, tc in L})
        for h in range(nh):
            wb += self.n * wavefronts({l: mi * self.region + 16 * self.chunk(h, tc) for l, mi, tr, tc in L})
        return wa, wb, ws

    def init_wavefronts(self, warp=0):
        """wavefronts of the one-time read of the staged (packed, row stride n)
        matrix into the accumulators; the write-back costs the same.  Rows of
        whole 16-B chunks: run_f32t's rotated 16-B accesses (PVEC); else 4-B
        element accesses (a 32-bit access costs its largest number of distinct
        addresses in one bank)."""
        L = self.lanes(warp)
        nh = self.cb // self.vec
        tot = 0
        for i in range(self.ra):
            if (self.n * self.es) % 16 == 0:
                for st in range(nh):
                    tot += wavefronts({l: mi * self.region + (self.row(i, tr) * self.n
                                                              + self.chunk((st + tr % nh) % nh, tc) * self.vec) * self.es
                                       for l, mi, tr, tc in L})
            else:
                for e in range(self.cb):
                    banks = {}
                    for l, mi, tr, tc in L:
                        a = mi * self.region + (self.row(i, tr) * self.n + self.chunk(e // self.vec, tc) * self.vec
                                                + e % self.vec) * self.es
                        banks.setdefault((a // 4) % 32, set()).add(a)
                    tot += max(len(v) for v in banks.values())
        return tot

    def score(self, maxreg=128):
        wa, wb, ws = self.update_wavefronts()
        # FMA-pipe clocks per update (SM-wide): FP32 2 FFMA2 / clk, FP64 2 DFMA / clk (64 FMA/clk/SM)
        fclk = (self.ra * self.cb // 2 * self.n) / 2.0 if self.es == 4 else (self.ra * self.cb * self.n) / 2.0
        # the one-time read + write-back, per update at the repeat count scored for
        # (STREAM: R = 1; resident: R = 100)
        wi = 2 * self.init_wavefronts() / (1 if STREAM else 100)
        lsu = (wa + wb + ws + wi) / fclk                   # LSU clocks per FMA clock
        live = len(self.lanes(0)) / 32.0
        pad = self.n * self.n / (self.nr * self.nc)
        regs = self.regs
        wps = 4 if regs <= 128 else (3 if regs <= 168 else 2)      # warps per SMSP from registers
        mats_sm = (227 * 1024) // (self.region * (2 if STREAM else 1))   # the streaming kernel double-buffers
        warps_sm_smem = mats_sm * self.wpm // self.mpw if self.wpm > 1 else mats_sm // self.mpw
        wps = min(wps, warps_sm_smem // 4)
        # FP32 pipe vs the register-file return of shared loads (microbench
        # ffma2_lds_mix: 8x8 0.81, 8x12 0.85, 8x16 0.87 with A one k ahead;
        # the per-row A block (at = 0) measured 0.77 at 8x8)
        ratio = 4.0 * (self.ra + self.cb) / (self.ra * self.cb)
        core = 1.0 / (1.0 + 0.30 * ratio)
        occ = {0: 0.0, 1: 0.7, 2: 0.95}.get(wps, 1.0)
        eff = pad * live * occ * core * min(1.0, 0.8 / lsu) if lsu > 0 else 0.0
        return {"eff": eff, "pad": pad, "live": live, "lsu": lsu, "wps": wps, "regs": regs,
                "wf": (wa, wb, ws), "region": self.region}


RA_MAX, CB_MAX = 8, 16   # r02 extended search: tools/f32_search.py --wide sets 13 / 24
STREAM = False           # score for the low-repeat kernel (two regions per matrix in flight)


def candidates(n, maxreg=128, es=4):
    vec = 16 // es
    for ra in range(2, RA_MAX + 1):
        for cb in range(vec, CB_MAX + 1, vec):
            rg, cg = cdiv(n, ra), cdiv(n, cb)
            t = rg * cg
            if t > 64 or (es // 4) * (ra * cb + vec * ra + 2 * cb) + 14 > 240:
                continue
            nc = cg * cb
            for ldmpad in range(1, 9):
                for pad in range(0, 8):
                    for colblk in (0, 1):
                        if cg == 1 and colblk:
                            continue
                        for trfast in (1, 0):
                            for qmix in ((0, 1) if 8 < t <= 16 else (0,)):
                                yield Cand(n, ra, cb, rg, cg, nc + vec * ldmpad, pad, colblk, trfast, qmix, es)


def best_for(n, top=5, maxreg=128, es=4):
    scored = []
    seen = set()
    for c in candidates(n, maxreg, es):
        s = c.score(maxreg)
        key = (c.ra, c.cb)
        scored.append((s["eff"], -s["region"], c, s))
    scored.sort(key=lambda x: (x[0], x[1]), reverse=True)
    out = []
    for e, _, c, s in scored:
        key = (c.ra, c.cb)
        if key in seen:
            continue
        seen.add(key)
        out.append((c, s))
        if len(out) >= top:
            break
    return out


def defines_for(n, ra, cb):
    """JM_BUILD_DEFINES forcing the best layout (under the model) of one FP32 shape."""
    best = None
    for c in candidates(n):
        if (c.ra, c.cb) != (ra, cb):
            continue
        s = c.score()
        if best is None or s["eff"] > best[1]["eff"]:
            best = (c, s)
    c = best[0]
    return (f"JM_F32T_RA={c.ra} JM_F32T_CB={c.cb} JM_F32T_LDMPAD={(c.ldm - c.nc) // 4} JM_F32T_PAD={c.pad} "
            f"JM_F32T_COLBLK={c.colblk} JM_F32T_TRFAST={c.trfast} JM_F32T_QMIX={c.qmix}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", default="17..64")
    ap.add_argument("--top", type=int, default=3)
    ap.add_argument("--emit", action="store_true")
    ap.add_argument("--defines", default=None, help="RAxCB -> JM_BUILD_DEFINES of its best FP32 layout")
    a = ap.parse_args()
    if a.defines:
        ra, cb = map(int, a.defines.split("x"))
        print(defines_for(int(a.n), ra, cb))
        return
    lo, _, hi = a.n.partition("..")
    ns = range(int(lo), int(hi or lo) + 1)
    rows = []
    from multiprocessing import Pool
    with Pool() as pool:
        results = pool.starmap(best_for, [(n, a.top) for n in ns])
    for n, res in zip(ns, results):
        rows.append((n, res[0][0]))
        if not a.emit:
            for c, s in res:
                print(f"n={n} {c.ra}x{c.cb} ({c.rg}x{c.cg}={c.tpmat} thr) ldm={c.ldm} pad={c.pad} colblk={c.colblk} "
                      f"trfast={c.trfast} qmix={c.qmix} "
                      f"eff={s['eff']:.3f} pad={s['pad']:.2f} live={s['live']:.2f} lsu={s['lsu']:.2f} "
                      f"wps={s['wps']} regs~{s['regs']} wf(A,B,S)={s['wf']} region={s['region']}")
    if a.emit:
        for n, c in rows:
            print(f"    {{{n}, {c.ra}, {c.cb}, {(c.ldm - c.cg * c.cb) // c.vec}, {c.pad}, {c.colblk}, {c.trfast}, "
                  f"{c.qmix}}},  // regs~{c.regs}")


if __name__ == "__main__":
    main()
