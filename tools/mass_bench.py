#!/usr/bin/env python3
"""Laghos mass-action benchmark — the B200 analog of PAPER.md Fig. 7.

Fig. 7 times rMassMultAdd2D<dofs, quads> on 10,000 elements, JIT-specialized vs
non-specialized (speedups 2.2-8.1x).  Here: jit_mat_mass specialized
(NVRTC k_mass<D, Q>) vs generic (runtime D, Q) at the figure's (d, q) pairs,
on 10,000 elements (the paper's size; latency-bound on a B200) and on 2^21
elements (HBM-bound), with the achieved HBM fraction.

    python tools/mass_bench.py [--out gpurun_out/mass.jsonl]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1904_08555_b200 as jm  # noqa: E402

HBM = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
PAIRS = [(2, 4), (2, 2), (4, 8), (2, 8), (4, 2), (4, 4), (8, 4), (8, 2), (8, 8)]


def timed(fn, steps, stream):
    fn()
    stream.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        fn()
    e1.record(stream)
    e1.synchronize()
    return e0.elapsed_time(e1) / steps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--pairs", default="fig7", help="fig7 (the figure's (d, q)) or all (1..8 x 1..8)")
    ap.add_argument("--elements", default="10000,2097152")
    a = ap.parse_args()
    pairs = PAIRS if a.pairs == "fig7" else [(d, q) for d in range(1, 9) for q in range(1, 9)]
    fh = open(a.out, "a") if a.out else None
    torch.cuda.init()
    jm.jit_mat_init(0)
    stream = torch.cuda.Stream()
    for D, Q in pairs:
        for E in map(int, a.elements.split(",")):
            B = torch.rand(Q, D, dtype=torch.float64, device="cuda")
            op = torch.rand(E, Q, Q, dtype=torch.float64, device="cuda") + 0.5
            x = torch.rand(E, D, D, dtype=torch.float64, device="cuda")
            y = torch.zeros(E, D, D, dtype=torch.float64, device="cuda")
            row = {"config": "F7-analog", "dofs": D, "quads": Q, "elements": E}
            for kind in ("specialized", "generic"):
                def call():
                    jm.jit_mat_mass(D, Q, E, B.data_ptr(), op.data_ptr(), x.data_ptr(), y.data_ptr(),
                                    kind=kind, stream=stream.cuda_stream)
                ms = timed(call, 20 if E > 10_000 else 200, stream)
                byts = E * (3 * D * D + Q * Q) * 8
                flops = E * (4 * D * Q * (D + Q) + Q * Q)
                row[kind] = {"ms": ms, "elements_per_s": E / (ms * 1e-3), "hbm_gbs": byts / (ms * 1e-3) / 1e9,
                             "frac_hbm": byts / (ms * 1e-3) / 1e9 / HBM, "gflops": flops / (ms * 1e-3) / 1e9}
            row["specialized_speedup"] = row["generic"]["ms"] / row["specialized"]["ms"]
            s = json.dumps(row)
            print(s, flush=True)
            if fh:
                fh.write(s + "\n")
            del B, op, x, y
    torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
