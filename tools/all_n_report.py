#!/usr/bin/env python3
"""Render an all-n sweep (tools/stream_sweep.py --sizes 2..64 --dtypes f64,f32
--repeats 1,100) as the markdown table under profiles/, optionally beside an
earlier sweep.

    python tools/all_n_report.py profiles/r02_all_n_sweep.jsonl [--before profiles/r01_all_n_sweep.jsonl]

R = 1 is reported against HBM where R(n+1) < 46, else against
the pipe (compute-bound even at one update); R = 100 against the pipe.
"""
from __future__ import annotations

import argparse
import json
import statistics


def load(path):
    t = {}
    for ln in open(path):
        d = json.loads(ln)
        n, R = d["n"], d["repeat"]
        hbm = R * (n + 1) < 46
        f = d["auto"]["frac_hbm" if hbm else "frac_pipe"]
        tile = d["kernels"].get(str(d["auto"]["variant"]), {}).get("tile", "?")
        t[(n, d["dtype"], R)] = (f, "HBM" if hbm else "pipe", tile)
    return t


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("path")
    ap.add_argument("--before", default=None)
    a = ap.parse_args()
    t = load(a.path)
    b = load(a.before) if a.before else {}
    print(f"# Every n = 2..64, FP64 and FP32, R = 1 and R = 100 — `{a.path.split('/')[-1]}` (one B200)\n")
    print("`python tools/stream_sweep.py --sizes 2..64 --dtypes f64,f32 --repeats 1,100 --gb 0.5`: the kernel the "
          "library picks, input 0.5 GB per config (> L2). R = 1: fraction of HBM (MEASURED_PEAKS.json) where "
          "R(n+1) < 46, else of the pipe (marked `p`: compute-bound even at one update); R = 100: fraction of "
          "the FP64 37.2 / FP32 74.4 TF pipe. "
          + (f"In brackets: `{a.before.split('/')[-1]}`." if b else "") + "\n")
    print("| n | f64 R=1 | f64 R=100 | f64 kernel (R=100 / R=1) | f32 R=1 | f32 R=100 | f32 kernel (R=100 / R=1) |")
    print("|---|---|---|---|---|---|---|")

    def cell(k):
        f, roof, _ = t[k]
        s = f"{f:.2f}" + ("p" if roof == "pipe" and k[2] == 1 else "")
        if k in b:
            s += f" ({b[k][0]:.2f})"
        return s
    for n in range(2, 65):
        row = [str(n)]
        for dt in ("f64", "f32"):
            row += [cell((n, dt, 1)), cell((n, dt, 100)), f"{t[(n, dt, 100)][2]} / {t[(n, dt, 1)][2]}"]
        print("| " + " | ".join(row) + " |")
    print()
    for dt in ("f64", "f32"):
        for R in (1, 100):
            v = [t[(n, dt, R)][0] for n in range(2, 65)]
            print(f"* {dt} R = {R}: median {statistics.median(v):.2f}, min {min(v):.2f} (n = "
                  f"{min(range(2, 65), key=lambda n: t[(n, dt, R)][0])})")


if __name__ == "__main__":
    main()
