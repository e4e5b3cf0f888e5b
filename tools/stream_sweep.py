#!/usr/bin/env python3
"""Resident vs streaming variant of the specialized update at low repeat -> JSON lines.

    python tools/stream_sweep.py [--sizes 8,16,32,64] [--dtypes f64,f32] [--repeats 1,2,4,8]

For each (n, dtype) a batch of ~`--gb` GB of input (> L2) is filled on the
device; each repeat count is timed with CUDA events on the launch stream for
both variants (forced through JM_FLAG_RESIDENT / JM_FLAG_STREAMING) and for
the library's own choice.  Fractions are of the measured HBM bandwidth
(MEASURED_PEAKS.json) and of the nominal FP64 / FP32 pipe.
Used to place the switch point (jm_plan.h JM_STREAM_RN).
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
PEAK = {"f64": 148 * 64 * 2 * 1.965e9 / 1e12, "f32": 148 * 128 * 2 * 1.965e9 / 1e12}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="8,12,16,17,24,32,40,48,64")
    ap.add_argument("--dtypes", default="f64,f32")
    ap.add_argument("--repeats", default="1,2,4,8")
    ap.add_argument("--gb", type=float, default=4.0)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    torch.cuda.init()
    jm.jit_mat_init(0)
    st = torch.cuda.Stream()
    fh = open(a.out, "a") if a.out else None
    flags = {"resident": jm.JM_FLAG_RESIDENT, "streaming": jm.JM_FLAG_STREAMING, "auto": 0}
    for dt in a.dtypes.split(","):
        es = 8 if dt == "f64" else 4
        tdt = torch.float64 if dt == "f64" else torch.float32
        sizes = []
        for part in a.sizes.split(","):      # "8,16" or ranges "2..64"
            lo, _, hi = part.partition("..")
            sizes += range(int(lo), int(hi or lo) + 1)
        for n in sizes:
            B = int(a.gb * 1e9 // (n * n * es))
            x = torch.empty(B, n, n, dtype=tdt, device="cuda")
            y = torch.empty_like(x)
            jm.jit_mat_fill(n, dt, 1, 0x0019040855, 0, B, x.data_ptr())
            torch.cuda.synchronize()
            for R in map(int, a.repeats.split(",")):
                row = {"n": n, "dtype": dt, "batch": B, "repeat": R}
                for name, fl in flags.items():
                    v = jm.jit_mat_prepare_for(n, dt, R, flags=fl)
                    run = lambda: jm.jit_mat_run_ex(n, dt, B, R, x.data_ptr(), y.data_ptr(),  # noqa: E731
                                                    stream=st.cuda_stream, flags=fl)
                    for _ in range(2):
                        run()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(st)
                    for _ in range(a.steps):
                        run()
                    e1.record(st)
                    e1.synchronize()
                    ms = e0.elapsed_time(e1) / a.steps
                    gbs = 2 * B * n * n * es / (ms / 1e3) / 1e9
                    tf = B * R * (2 * n ** 3 + 2 * n * n) / (ms / 1e3) / 1e12
                    row[name] = {"variant": v, "ms": round(ms, 4), "hbm_gbs": round(gbs, 1),
                                 "frac_hbm": round(gbs / HBM, 3), "frac_pipe": round(tf / PEAK[dt], 3)}
                info = {k["variant"]: k for k in jm.jit_mat_key_info()
                        if k["op"] == 0 and k["n"] == n and k["dtype"] == (1 if dt == "f64" else 0)
                        and k["kind"] == 0 and k["addend"] == 0}
                row["kernels"] = {str(v): {"regs": k["regs"], "smem": k["smem_bytes"], "local": k["local_bytes"],
                                           "tile": k["tile_name"]} for v, k in info.items()}
                s = json.dumps(row)
                print(s, flush=True)
                if fh:
                    fh.write(s + "\n")
                    fh.flush()
            del x, y
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
