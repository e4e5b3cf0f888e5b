#!/usr/bin/env python3
"""The configuration list of the per-kind ncu capture (VERDICT r01 "one committed
ncu summary per shipping kernel kind"): one launch of every tiling kind the
planner ships, each variant (resident / streaming / latency), both dtypes.

    python tools/ncu_kinds.py            -> the n:dtype:batch:repeat:variant specs (tools/ncu_configs.py)
    python tools/ncu_kinds.py --algo     -> the matching n,dtype,batch,repeat list (tools/ncu_summary.py --algo)

Batches hold ~0.5 GB of input (> L2) except the latency kernel (batch 1).
"""
from __future__ import annotations

import sys

# (what, n, dtype, repeat, variant)
KINDS = [
    ("TPM f64 (thread per matrix), HBM side", 2, "f64", 1, "auto"),
    ("TPM f64, HBM side", 4, "f64", 1, "auto"),
    ("TPM f64, FP64 side", 4, "f64", 100, "auto"),
    ("TPM f32 (FFMA2), HBM side", 4, "f32", 1, "auto"),
    ("TPM f32 with prefetching stage", 8, "f32", 100, "auto"),
    ("TPMS f64 (staged product)", 10, "f64", 100, "auto"),
    ("TPMS f32 (staged product)", 13, "f32", 100, "auto"),
    ("F64 register tiles (DFMA)", 12, "f64", 100, "auto"),
    ("F64 register tiles (DFMA)", 20, "f64", 100, "auto"),
    ("DMMA ring (low-repeat kernel of the register-tile sizes)", 20, "f64", 1, "auto"),
    ("warp DMMA (C2)", 16, "f64", 100, "auto"),
    ("warp DMMA, HBM side (resident)", 16, "f64", 1, "auto"),
    ("F64 register tiles (DFMA), 9 x 6", 17, "f64", 100, "auto"),
    ("warp DMMA + thin border", 25, "f64", 100, "auto"),
    ("warp DMMA + k-compaction", 28, "f64", 100, "auto"),
    ("warp DMMA, whole matrix per warp", 40, "f64", 100, "auto"),
    ("DMMA ring (streaming), warp per matrix", 32, "f64", 1, "auto"),
    ("CTA DMMA", 48, "f64", 100, "auto"),
    ("CTA DMMA", 64, "f64", 100, "auto"),
    ("CTA DMMA ring (streaming)", 40, "f64", 1, "auto"),
    ("CTA DMMA ring (streaming)", 64, "f64", 1, "auto"),
    ("F32 row panels", 15, "f32", 100, "auto"),
    ("F32 row-panel ring (streaming)", 15, "f32", 1, "auto"),
    ("F32 tiles, resident kernel", 16, "f32", 100, "resident"),
    ("F32 tile ring (streaming), 8 x 4", 16, "f32", 1, "streaming"),
    ("F32 tiles, resident kernel", 17, "f32", 100, "resident"),
    ("F32 tiles, resident kernel", 24, "f32", 100, "resident"),
    ("F32 tiles, resident kernel", 32, "f32", 100, "resident"),
    ("F32 tiles, resident kernel", 48, "f32", 100, "resident"),
    ("F32 tiles, resident kernel", 64, "f32", 100, "resident"),
    ("F32 tiles, streaming kernel at R = 100 (its pick: two-warp 8x8 shape)", 32, "f32", 100, "streaming"),
    ("F32 tiles, streaming kernel (prefetching stage, odd n)", 17, "f32", 1, "streaming"),
    ("F32 tile ring (streaming, even n)", 24, "f32", 1, "streaming"),
    ("F32 tile ring (streaming, even n)", 32, "f32", 1, "streaming"),
    ("F32 tiles, prefetching stage (streaming, odd n)", 33, "f32", 1, "streaming"),
    ("F32 tile ring (streaming, even n)", 48, "f32", 1, "streaming"),
    ("F32 tiles, streaming kernel (compute-bound at R = 1)", 64, "f32", 1, "streaming"),
    ("latency kernel (C1: one 4x4, warp per matrix)", 4, "f64", 1000, "latency"),
    ("generic runtime-N kernel", 16, "f64", 100, "generic"),
]


def batch(n, dt, variant):
    if variant == "latency":
        return 1
    es = 8 if dt == "f64" else 4
    return int(0.5e9 // (n * n * es))


def main():
    if "--algo" in sys.argv:
        print(" ".join(f"{n},{dt},{batch(n, dt, v)},{r}" for _, n, dt, r, v in KINDS))
    elif "--what" in sys.argv:
        for w, n, dt, r, v in KINDS:
            print(f"{w}\t{n}\t{dt}\tR={r}\t{v}")
    else:
        print(" ".join(f"{n}:{dt}:{batch(n, dt, v)}:{r}:{v}" for _, n, dt, r, v in KINDS))


if __name__ == "__main__":
    main()
