#!/usr/bin/env python3
"""Measured per-n choice of the register-tile configuration (run_f32t / run_f64t,
jm_plan.h F32T_TABLE / F64T_TABLE).

    python tools/f32_search.py --candidates 17..64 > tools/f32_candidates.json   (CPU: layout model)
    python tools/f32_search.py --run tools/f32_candidates.json --out R.jsonl      (GPU box)
    python tools/f32_search.py --pick R.jsonl                                     (-> table rows)

--candidates ranks, per n, the register tiles of tools/f32_layout.py (each
with its best layout) and attaches a register cap and k-loop unrolling.
--run writes the j-th candidate of every n into jm_plan.h's table (of the
scratch copy on the GPU box), rebuilds, and times every n at R = 100 with
tools/stream_sweep.py, for j = 0, 1, ...; --pick keeps the fastest per n.
"""
from __future__ import annotations

import argparse
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PLAN = os.path.join(ROOT, "paper_1904_08555_b200", "csrc", "kernels", "jm_plan.h")
sys.path.insert(0, os.path.join(ROOT, "tools"))


def row(c: dict) -> str:
    wpc = f", {c['wpc']}" if c.get("wpc") else ""
    return (f"    {{{c['n']}, {c['ra']}, {c['cb']}, {c['ldmpad']}, {c['pad']}, {c['colblk']}, {c['trfast']}, "
            f"{c['qmix']}, {c['maxreg']}, {c['kunroll']}{wpc}}},")


def write_table(rows: list[str], dt: str = "f32", stream: bool = False) -> None:
    name = "F32TS_TABLE" if stream else "F32T_TABLE" if dt == "f32" else "F64T_TABLE"
    s = open(PLAN).read()
    a = s.index(f"constexpr F32TRow {name}[] = {{")
    b = s.index("};", a)
    body = "\n".join(rows) if rows else "    {0, 0, 0, 0, 0, 0, 0, 0, 0, 0},"
    s = s[:a] + f"constexpr F32TRow {name}[] = {{\n" + body + "\n" + s[b:]
    open(PLAN, "w").write(s)


def candidates(ns, top, es=4, wide=False, stream=False):
    import f32_layout as L
    if wide:   # r02: register tiles up to 12 (FP64) / 13 (FP32) rows and 12 / 24 columns
        L.RA_MAX, L.CB_MAX = (12, 12) if es == 8 else (13, 24)
    L.STREAM = stream
    from multiprocessing import Pool
    with Pool(initializer=_widen, initargs=(L.RA_MAX, L.CB_MAX, L.STREAM)) as pool:
        res = pool.starmap(L.best_for, [(n, top, 128, es) for n in ns])
    out = {}
    for n, lst in zip(ns, res):
        cs = []
        for c, s in lst:
            regs = c.regs
            base = dict(n=n, ra=c.ra, cb=c.cb, ldmpad=(c.ldm - c.nc) // c.vec, pad=c.pad, colblk=c.colblk,
                        trfast=c.trfast, qmix=c.qmix, model_eff=round(s["eff"], 3), regs_est=regs)
            ku_full = max(1, n // c.vec)
            cs.append(dict(base, maxreg=168 if regs + 10 <= 168 else 255, kunroll=ku_full if n <= 48 else 2))
            cs.append(dict(base, maxreg=255, kunroll=2))
        out[n] = cs
    return out


def _widen(ra_max, cb_max, stream=False):
    import f32_layout as L
    L.RA_MAX, L.CB_MAX, L.STREAM = ra_max, cb_max, stream


def run(cands: dict, out: str, steps: int, dt: str = "f32", baseline: bool = False, stream: bool = False) -> None:
    """stream: the candidates go into F32TS_TABLE (the low-repeat kernel's own
    shapes) and are timed at R = 1 (fraction of HBM, the library's pick)"""
    ns = sorted(int(n) for n in cands)
    depth = max(len(v) for v in cands.values())
    for j in ([-1] if baseline else []) + list(range(depth)):
        # rank -1: the table empty (FP64: the DMMA / TPMS kinds these sizes use otherwise)
        rows = [] if j < 0 else [row(cands[str(n)][min(j, len(cands[str(n)]) - 1)]) for n in ns]
        write_table(rows, dt, stream)
        b = subprocess.run([sys.executable, "-c", "import paper_1904_08555_b200._build as b; b.build(force=True)"],
                           cwd=ROOT, capture_output=True, text=True)
        if b.returncode:
            print(f"rank {j}: build failed: {b.stderr[-2000:]}", file=sys.stderr)
            continue
        p = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "stream_sweep.py"), "--sizes",
                            ",".join(map(str, ns)), "--dtypes", dt, "--repeats", "1" if stream else "100",
                            "--gb", "0.5" if stream else "0.25",
                            "--steps", str(steps)], cwd=ROOT, capture_output=True, text=True)
        with open(out, "a") as fh:
            for ln in p.stdout.splitlines():
                d = json.loads(ln)
                n = d["n"]
                c = None if j < 0 else cands[str(n)][min(j, len(cands[str(n)]) - 1)]
                k = d["kernels"]["1" if stream else "0"]
                frac = d["auto"]["frac_hbm"] if stream else d["resident"]["frac_pipe"]
                rec = dict(rank=j, n=n, dtype=dt, cand=c, frac_pipe=frac, regs=k["regs"],
                           local=k["local"], smem=k["smem"], tile=k["tile"], stream=stream)
                fh.write(json.dumps(rec) + "\n")
        print(f"rank {j} done", file=sys.stderr)


def pick(path: str, margin: float = 0.0) -> None:
    """Fastest candidate per n; with a baseline (rank -1) only sizes the
    register tiles beat by more than `margin` are emitted."""
    best, base = {}, {}
    for ln in open(path):
        d = json.loads(ln)
        n = d.get("n") or d["cand"]["n"]
        if d["rank"] < 0:
            base[n] = d["frac_pipe"]
            continue
        if d["local"] > 0:
            continue
        if n not in best or d["frac_pipe"] > best[n]["frac_pipe"]:
            best[n] = d
    for n in sorted(best):
        b = best[n]
        if n in base and b["frac_pipe"] <= base[n] + margin:
            print(f"    // n = {n}: register tiles {b['frac_pipe']:.3f} vs {base[n]:.3f} without: not taken")
            continue
        extra = f" (was {base[n]:.3f})" if n in base else ""
        print(row(b["cand"]) + f"  // {b['frac_pipe']:.3f} of the pipe{extra}, {b['regs']} regs")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--candidates", default=None)
    ap.add_argument("--top", type=int, default=3)
    ap.add_argument("--run", default=None)
    ap.add_argument("--out", default="f32_search.jsonl")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--pick", default=None)
    ap.add_argument("--dtype", default="f32", choices=["f32", "f64"])
    ap.add_argument("--baseline", action="store_true", help="also time the sizes with the table empty")
    ap.add_argument("--margin", type=float, default=0.0)
    ap.add_argument("--wide", action="store_true", help="larger register tiles (see candidates())")
    ap.add_argument("--stream", action="store_true", help="search the low-repeat kernel's table (R = 1, HBM)")
    a = ap.parse_args()
    if a.candidates:
        ns = []
        for part in a.candidates.split(","):
            lo, _, hi = part.partition("..")
            ns += list(range(int(lo), int(hi or lo) + 1))
        print(json.dumps(candidates(ns, a.top, 8 if a.dtype == "f64" else 4, a.wide, a.stream), indent=0))
    elif a.run:
        run(json.load(open(a.run)), a.out, a.steps, a.dtype, a.baseline, a.stream)
    elif a.pick:
        pick(a.pick, a.margin)


if __name__ == "__main__":
    main()
