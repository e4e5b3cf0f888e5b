#!/usr/bin/env python3
"""Small invocation of every kernel kind, for compute-sanitizer.

    compute-sanitizer --tool memcheck  python tools/sanitize_run.py
    compute-sanitizer --tool racecheck python tools/sanitize_run.py
    compute-sanitizer --tool synccheck python tools/sanitize_run.py

Covers TPM, warp/CTA DMMA (incl. the thin-border sizes), FP32 row panels and
tiles, each in its resident and streaming (bulk-copy ring) variant, the generic kernels, the
AoT specializations, the multiply-accumulate, fill, checksum, run_many and the
host-buffer path, the mass action (both kernels), each on a ragged batch (several chunks + a partial one).
Exits non-zero on any library error; the sanitizer reports the rest.
"""
from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1904_08555_b200 as jm  # noqa: E402

# r02 adds: the FP64 register tiles (11, 17, 20) and their DMMA ring, k-compaction (28, 44),
# the thin border (25), FP32 tiles with their own streaming shapes, two-warp CTAs, the
# rotated 16-B one-time accesses (20, 32, 48, 64) and the prefetching stage (odd n: 21, 49)
CASES = [(2, "f64"), (3, "f64"), (5, "f64"), (7, "f64"), (9, "f64"), (10, "f64"), (16, "f64"),
         (11, "f64"), (13, "f64"), (17, "f64"), (20, "f64"), (25, "f64"), (26, "f64"), (28, "f64"),
         (32, "f64"), (33, "f64"), (40, "f64"), (44, "f64"), (48, "f64"), (64, "f64"),
         (3, "f32"), (8, "f32"), (10, "f32"), (12, "f32"), (13, "f32"), (16, "f32"), (17, "f32"),
         (20, "f32"), (21, "f32"), (24, "f32"), (32, "f32"), (33, "f32"), (48, "f32"), (49, "f32"),
         (53, "f32"), (64, "f32")]


def main():
    torch.cuda.init()
    jm.jit_mat_init(0)
    for n, dt in CASES:
        tdt = torch.float64 if dt == "f64" else torch.float32
        batch = 37 if n <= 16 else 5
        x = torch.empty(batch, n, n, dtype=tdt, device="cuda")
        jm.jit_mat_fill(n, dt, 2, 7, 0, batch, x.data_ptr())
        for kind in ("specialized", "generic"):
            for addend in ("ones", "identity"):
                jm.run(x, 2, addend=addend, kind=kind, sync=True)
        for variant in ("resident", "streaming"):      # both variants where the kind has two
            jm.run(x, 2, variant=variant, sync=True)
            jm.run(x.clone(), 1, variant=variant, sync=True)
        y = x.clone()
        jm.run(y, 2, y, sync=True)                       # in place
        jm.jit_mat_checksum(n, dt, 0, batch, y.data_ptr())
        c = torch.zeros_like(x)
        jm.matmul(x, x, c, sync=True)
        jm.matmul(x, x, c, kind="generic", sync=True)
        print(f"ok n={n} {dt}", flush=True)
    # streaming ring with several chunks per CTA (refills behind bulk stores)
    for n, dt, b in ((16, "f64", 4741), (33, "f64", 700), (20, "f32", 3001)):
        tdt = torch.float64 if dt == "f64" else torch.float32
        x = torch.rand(b, n, n, dtype=tdt, device="cuda")
        jm.run(x, 1, variant="streaming", sync=True)
        print(f"ok ring n={n} {dt} batch={b}", flush=True)
    x = torch.rand(11, 16, 16, dtype=torch.float64, device="cuda")
    jm.run(x, 3, kind="aot_specialized", sync=True)
    for n in (2, 4, 5):   # the latency kernel (a warp per matrix, tiny batches)
        x = torch.rand(3, n, n, dtype=torch.float64, device="cuda")
        jm.run(x, 5, variant="latency", sync=True)
    groups = []
    bufs = []
    for n in (2, 9, 17, 40):
        a = torch.rand(6, n, n, dtype=torch.float64, device="cuda")
        b = torch.empty_like(a)
        bufs.append((a, b))
        groups.append(dict(n=n, dtype="f64", batch=6, repeat=2, in_ptr=a.data_ptr(), out_ptr=b.data_ptr()))
    jm.jit_mat_run_many(groups, sync=True)
    # Laghos mass action: thread-per-element (4, 4), (3, 5) and the r02 DMMA kernel (8, 8), (8, 3), (2, 8),
    # ragged element counts (a partial CTA chunk; fewer elements than warps)
    for D, Q, E in ((4, 4, 301), (3, 5, 77), (8, 8, 301), (8, 3, 5), (2, 8, 1029)):
        B = torch.rand(Q, D, dtype=torch.float64, device="cuda")
        op = torch.rand(E, Q, Q, dtype=torch.float64, device="cuda")
        xm = torch.rand(E, D, D, dtype=torch.float64, device="cuda")
        ym = torch.rand(E, D, D, dtype=torch.float64, device="cuda")
        for kind in ("specialized", "generic"):
            jm.mass(B, op, xm, ym, kind=kind, sync=True)
    h = np.random.default_rng(0).random((300, 4, 4))
    out = np.empty_like(h)
    os.environ["JIT_MAT_HOST_CHUNK_MB"] = "0"
    jm.jit_mat_run_host(4, "f64", 300, 2, h.ctypes.data, out.ctypes.data)
    torch.cuda.synchronize()
    print("sanitize_run: all kinds exercised")


if __name__ == "__main__":
    main()
