#!/usr/bin/env python3
"""Render a mass-action A/B (tools/ab.py --tool mass_bench: every (D, Q) in
1..8 x 1..8 at 2^21 elements, one JSON line per pair and variant) as a table
of HBM fractions per variant, plus the pairs where each variant wins.

    python tools/mass_report.py gpurun_out/mass_ab.jsonl [--pick thread,dmma_pd4]
"""
from __future__ import annotations

import argparse
import json
import statistics


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("path")
    ap.add_argument("--pick", default=None, help="two variants: print the per-D bitmask where the second wins")
    a = ap.parse_args()
    t, names = {}, []
    for ln in open(a.path):
        d = json.loads(ln)
        if d["ab"] not in names:
            names.append(d["ab"])
        t.setdefault((d["dofs"], d["quads"]), {})[d["ab"]] = d["specialized"]["frac_hbm"]
    print("Fraction of HBM (MEASURED_PEAKS.json), specialized kernel, 2^21 elements; cells: "
          + " / ".join(names) + "\n")
    print("| D \\ Q | " + " | ".join(str(q) for q in range(1, 9)) + " |")
    print("|---|" + "---|" * 8)
    for D in range(1, 9):
        cells = ["/".join(f"{t[(D, Q)].get(v, float('nan')):.2f}" for v in names) for Q in range(1, 9)]
        print(f"| {D} | " + " | ".join(cells) + " |")
    print()
    for v in names:
        xs = [t[k][v] for k in t if v in t[k]]
        print(f"* {v}: median {statistics.median(xs):.2f}, min {min(xs):.2f}")
    if a.pick:
        base, new = a.pick.split(",")
        masks = []
        for D in range(1, 9):
            m = 0
            for Q in range(1, 9):
                if t[(D, Q)][new] > t[(D, Q)][base]:
                    m |= 1 << (Q - 1)
            masks.append(hex(m))
        print(f"* pairs where {new} beats {base} (row D, bit Q-1): {masks}")


if __name__ == "__main__":
    main()
