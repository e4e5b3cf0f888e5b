#!/usr/bin/env python3
"""One launch of the specialized Laghos mass action per (D, Q), for an ncu capture.

    ncu --set full --clock-control none -k regex:k_mass -o gpurun_out/mass python tools/mass_ncu.py 8:8 4:4

Inputs: 2^21 elements (x, y, op > L2), B ~ U[0,1), op ~ U[0.5,1.5).
"""
from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1904_08555_b200 as jm  # noqa: E402


def main():
    torch.cuda.init()
    jm.jit_mat_init(0)
    E = 1 << 21
    for spec in sys.argv[1:] or ["8:8", "4:4"]:
        D, Q = map(int, spec.split(":"))
        B = torch.rand(Q, D, dtype=torch.float64, device="cuda")
        op = torch.rand(E, Q, Q, dtype=torch.float64, device="cuda") + 0.5
        x = torch.rand(E, D, D, dtype=torch.float64, device="cuda")
        y = torch.zeros(E, D, D, dtype=torch.float64, device="cuda")
        jm.mass(B, op, x, y, sync=True)
        print(f"mass D={D} Q={Q} E={E} bytes={E * (3 * D * D + Q * Q) * 8}", flush=True)
        del B, op, x, y
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
