#!/usr/bin/env python3
"""Batched multiply-accumulate benchmark — the B200 analog of PAPER.md Fig. 6.

The paper's RAJA benchmark (Listing 8) calls a JIT-specialized 4-deep loop
kernel `repeats / batch_size` times; per call it pays a lookup of the compiled
instantiation, so small batches expose the lookup cost (Fig. 6: b1i8 at 2x2 is
0.43x, larger batches > 1x).  Here one call = one jit_mat_matmul launch of
`batch` matrices (c[b] += a[b] @ b[b]); per call the library does its cache
lookup (row a1) plus a kernel launch.  Reported per (n, batch):

* us per call and matrices/s for the specialized and the generic kernel, with
  plain launches and with the calls captured into a CUDA graph and replayed
  (the B200 answer to per-call overhead);
* the in-library cache-hit cost (jit_mat_time_lookup);
* a large HBM-bound batch (2^24 matrices) against the measured HBM roofline.

    python tools/matmul_bench.py [--out gpurun_out/matmul.jsonl]
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


def emit(d, fh):
    s = json.dumps(d)
    print(s, flush=True)
    if fh:
        fh.write(s + "\n")


def per_call_us(fn, calls, stream):
    fn()
    stream.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(calls):
        fn()
    e1.record(stream)
    e1.synchronize()
    return e0.elapsed_time(e1) * 1e3 / calls


def graph_us(fn, calls_per_graph, replays, stream):
    fn()
    stream.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for _ in range(calls_per_graph):
            fn()
    with torch.cuda.stream(stream):   # replay() launches on the current stream
        g.replay()
        stream.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(replays):
            g.replay()
        e1.record(stream)
        e1.synchronize()
    return e0.elapsed_time(e1) * 1e3 / (calls_per_graph * replays)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--calls", type=int, default=4000)
    a = ap.parse_args()
    fh = open(a.out, "a") if a.out else None
    torch.cuda.init()
    jm.jit_mat_init(0)
    stream = torch.cuda.Stream()
    for n in (2, 8):
        jm.jit_mat_prepare(n, "double")
        hit_ns = jm.jit_mat_time_lookup(n, "double", iters=1_000_000)
        for batch in (10, 1000, 10000):
            x = [torch.randn(batch, n, n, dtype=torch.float64, device="cuda") for _ in range(3)]
            row = {"config": "F6-analog", "n": n, "dtype": "f64", "batch": batch,
                   "lookup_hit_ns": hit_ns}
            for kind in ("specialized", "generic"):
                jm.jit_mat_matmul(n, "f64", batch, x[0].data_ptr(), x[1].data_ptr(), x[2].data_ptr(),
                                  kind=kind, stream=stream.cuda_stream)

                def call():
                    jm.jit_mat_matmul(n, "f64", batch, x[0].data_ptr(), x[1].data_ptr(),
                                      x[2].data_ptr(), kind=kind, stream=stream.cuda_stream)

                us = per_call_us(call, a.calls, stream)
                gus = graph_us(call, 200, max(1, a.calls // 200), stream)
                row[kind] = {"us_per_call": us, "matrices_per_s": batch / (us * 1e-6),
                             "graph_us_per_call": gus, "graph_matrices_per_s": batch / (gus * 1e-6)}
            row["specialized_speedup"] = row["generic"]["us_per_call"] / row["specialized"]["us_per_call"]
            row["specialized_speedup_graph"] = (row["generic"]["graph_us_per_call"]
                                                / row["specialized"]["graph_us_per_call"])
            emit(row, fh)
        # large batch: HBM roofline (4 n^2 elements of traffic per matrix)
        big = 1 << 24 if n == 2 else 1 << 22
        x = [torch.randn(big, n, n, dtype=torch.float64, device="cuda") for _ in range(3)]
        res = {"config": "HBM", "n": n, "dtype": "f64", "batch": big}
        for kind in ("specialized", "generic"):
            def call():
                jm.jit_mat_matmul(n, "f64", big, x[0].data_ptr(), x[1].data_ptr(), x[2].data_ptr(),
                                  kind=kind, stream=stream.cuda_stream)
            us = per_call_us(call, 10, stream)
            gbs = 4 * big * n * n * 8 / (us * 1e-6) / 1e9
            res[kind] = {"ms": us / 1e3, "matrices_per_s": big / (us * 1e-6), "hbm_gbs": gbs,
                         "frac_hbm": gbs / HBM}
        emit(res, fh)
        del x
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
