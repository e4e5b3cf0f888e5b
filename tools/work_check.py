#!/usr/bin/env python3
"""Work-done check (SURVEY.md §4 T4, §8(d) "ncu evidence per kernel kind").

At R >= ~20 every output converges to the same fixed point (oracle pin O4), so
parity alone cannot prove the update was executed R times.  This tool counts,
with ncu, the floating-point FMA work each kernel kind actually executes:

    FP64: DFMA thread instructions + 256 x DMMA.8x8x4 warp instructions
    FP32: FFMA thread instructions + 2 x FFMA2 thread instructions

and divides it by the algorithmic count n^2 (n+1) * batch * R (Ones addend).
Kinds without padding must come out at exactly 1; padded kinds report their
padding factor (DMMA 8x8x4 granularity, FP32 register-tile shapes).

    python tools/work_check.py [--out profiles/r01_work_check.jsonl]   (runs ncu per config)
    python tools/work_check.py --child N DTYPE BATCH REPEAT VARIANT     (one launch, under ncu)
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

METRICS = ["sm__sass_thread_inst_executed_op_dfma_pred_on.sum",
           "sm__inst_executed_pipe_tensor_subpipe_dmma.sum",
           "sm__sass_thread_inst_executed_op_ffma_pred_on.sum",
           "sm__sass_thread_inst_executed_op_ffma2_pred_on.sum"]

# (n, dtype, variant, exact): exact = no padding in this kind, ratio must be 1
CONFIGS = [(2, "f64", "resident", True), (4, "f64", "resident", True), (7, "f64", "resident", True),
           (8, "f64", "resident", True), (16, "f64", "resident", True), (16, "f64", "streaming", True),
           (32, "f64", "resident", True), (32, "f64", "streaming", True), (64, "f64", "resident", True),
           (9, "f64", "resident", True), (10, "f64", "resident", True),
           # FP64 register tiles (r02): 12 and 20 tile exactly, 11 and 17 pad to 12 / 18
           (12, "f64", "resident", True), (20, "f64", "resident", True),
           (11, "f64", "resident", False), (17, "f64", "resident", False),
           # DMMA padding: thin border (25), k-compaction (28), CTA kind (41)
           (25, "f64", "resident", False), (28, "f64", "resident", False), (41, "f64", "resident", False),
           (2, "f32", "resident", True), (3, "f32", "resident", True), (8, "f32", "resident", True),
           (11, "f32", "resident", True), (12, "f32", "resident", True), (16, "f32", "resident", True),
           # FP32 register tiles (r02 shapes): 24, 32, 48, 64 tile exactly; 17 pads to 18 x 20
           (24, "f32", "resident", True), (32, "f32", "resident", True), (48, "f32", "resident", True),
           (64, "f32", "resident", True), (32, "f32", "streaming", True), (17, "f32", "resident", False)]


def child(n, dt, batch, repeat, variant):
    import torch

    import paper_1904_08555_b200 as jm
    torch.cuda.init()
    jm.jit_mat_init(0)
    tdt = torch.float64 if dt == "f64" else torch.float32
    x = torch.empty(batch, n, n, dtype=tdt, device="cuda")
    jm.jit_mat_fill(n, dt, 1, 0x0019040855, 0, batch, x.data_ptr())
    if variant == "generic":
        jm.run(x, repeat, sync=True, kind="generic")
    else:
        jm.run(x, repeat, sync=True, variant=variant)


def parse(csv_text):
    rows = list(csv.reader(io.StringIO(csv_text)))
    hi = [i for i, r in enumerate(rows) if "Metric Name" in r][0]
    h = rows[hi]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    tot = {m: 0.0 for m in METRICS}
    kernels = set()
    for r in rows[hi + 1:]:
        if len(r) <= vi or "k_update" not in r[ki]:
            continue
        kernels.add(r[ki].split("(")[0])
        m = r[mi]
        if m in tot:
            tot[m] += float(r[vi].replace(",", ""))
    return tot, sorted(kernels)


def instructions(n, dt, kind, batch, repeat):
    """Total warp instructions executed by the update kernel (specialized or generic)."""
    cmd = ["ncu", "--csv", "--metrics", "smsp__inst_executed.sum", "-k", "regex:k_update|jm_generic",
           sys.executable, os.path.abspath(__file__), "--child", str(n), dt, str(batch), str(repeat),
           "generic" if kind == "generic" else "resident"]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    rows = list(csv.reader(io.StringIO(p.stdout)))
    hi = [i for i, r in enumerate(rows) if "Metric Name" in r][0]
    h = rows[hi]
    vi, ki = h.index("Metric Value"), h.index("Kernel Name")
    return sum(float(r[vi].replace(",", "")) for r in rows[hi + 1:]
               if len(r) > vi and ("k_update" in r[ki] or "jm_generic" in r[ki]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--child", nargs=5, default=None)
    ap.add_argument("--out", default=None)
    ap.add_argument("--batch", type=int, default=2048)
    ap.add_argument("--repeat", type=int, default=5)
    a = ap.parse_args()
    if a.child:
        n, dt, b, r, v = a.child
        child(int(n), dt, int(b), int(r), v)
        return
    fh = open(a.out, "a") if a.out else None
    bad = 0
    for n, dt, variant, exact in CONFIGS:
        cmd = ["ncu", "--csv", "--metrics", ",".join(METRICS), "-k", "regex:k_update",
               sys.executable, os.path.abspath(__file__), "--child", str(n), dt, str(a.batch), str(a.repeat),
               variant]
        p = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
        tot, kernels = parse(p.stdout)
        alg = n * n * (n + 1) * a.batch * a.repeat
        if dt == "f64":
            done = tot[METRICS[0]] + 256.0 * tot[METRICS[1]]
        else:
            done = tot[METRICS[2]] + 2.0 * tot[METRICS[3]]
        ratio = done / alg
        ok = (abs(ratio - 1.0) < 1e-9) if exact else (ratio >= 1.0 - 1e-9)
        bad += not ok
        row = {"n": n, "dtype": dt, "variant": variant, "batch": a.batch, "repeat": a.repeat,
               "kernels": kernels, "algorithmic_fma": alg, "executed_fma": done, "ratio": ratio,
               "exact_kind": exact, "ok": ok, "counts": tot}
        s = json.dumps(row)
        print(s, flush=True)
        if fh:
            fh.write(s + "\n")
            fh.flush()
    # SPEC.md:617/645 "specialized executes less": warp instructions of the
    # specialized vs the generic runtime-N kernel on the same launch (Fig. 3 sizes)
    for n, dt in ((3, "f64"), (7, "f64"), (16, "f64"), (16, "f32"), (64, "f64")):
        spec = instructions(n, dt, "specialized", a.batch, a.repeat)
        gen = instructions(n, dt, "generic", a.batch, a.repeat)
        row = {"check": "instructions", "n": n, "dtype": dt, "batch": a.batch, "repeat": a.repeat,
               "specialized_warp_inst": spec, "generic_warp_inst": gen, "generic_over_specialized": gen / spec}
        bad += not (spec < gen)
        s = json.dumps(row)
        print(s, flush=True)
        if fh:
            fh.write(s + "\n")
            fh.flush()
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
