#!/usr/bin/env python3
"""Candidates around the current register-tile table rows (jm_plan.h) for
tools/f32_search.py --run: for each n, the shipped row with its register cap,
k-loop unrolling, warps per CTA and region padding varied.

    python tools/neighborhood.py --dtype f32 --sizes 17,25,49,50 > /tmp/nb.json
    python tools/neighborhood.py --table F32TS_TABLE --sizes 16..64 --maxreg cur,168,255 --kunroll 2,4,8 --wpc cur

(--maxreg / --wpc accept "cur" for the shipped value; sizes without a row are skipped.)
"""
from __future__ import annotations

import argparse
import itertools
import json
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PLAN = os.path.join(ROOT, "paper_1904_08555_b200", "csrc", "kernels", "jm_plan.h")
KEYS = ["n", "ra", "cb", "ldmpad", "pad", "colblk", "trfast", "qmix", "maxreg", "kunroll", "wpc"]


def table(name: str) -> dict:
    s = open(PLAN).read()
    a = s.index(f"constexpr F32TRow {name}[] = {{")
    body = s[a:s.index("};", a)]
    rows = {}
    for m in re.finditer(r"\{\s*(\d+(?:\s*,\s*\d+){9,10})\s*\}", body):
        v = [int(x) for x in m.group(1).split(",")]
        if v[0]:
            rows[v[0]] = dict(zip(KEYS, v + [0] * (11 - len(v))))
    return rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dtype", default="f32", choices=["f32", "f64"])
    ap.add_argument("--table", default=None, help="F32T_TABLE (default f32), F64T_TABLE (f64) or F32TS_TABLE")
    ap.add_argument("--sizes", required=True)
    ap.add_argument("--maxreg", default="168,200,232,255")
    ap.add_argument("--kunroll", default="1,2,4,8")
    ap.add_argument("--wpc", default="0,2")
    ap.add_argument("--pad", default="")
    a = ap.parse_args()
    cur = table(a.table or ("F64T_TABLE" if a.dtype == "f64" else "F32T_TABLE"))
    vec = 2 if a.dtype == "f64" else 4
    out = {}
    sizes = []
    for part in a.sizes.split(","):
        lo, _, hi = part.partition("..")
        sizes += range(int(lo), int(hi or lo) + 1)
    for n in sizes:
        if n not in cur:
            continue
        base = cur[n]
        pads = [int(x) for x in a.pad.split(",")] if a.pad else [base["pad"]]
        cs = [dict(base, current=True)]
        val = lambda v, k: base[k] if v == "cur" else int(v)   # noqa: E731
        for mr, ku, wpc, pad in itertools.product([val(v, "maxreg") for v in a.maxreg.split(",")],
                                                  map(int, a.kunroll.split(",")),
                                                  [val(v, "wpc") for v in a.wpc.split(",")], pads):
            ku = min(ku, max(1, n // vec))
            c = dict(base, maxreg=mr, kunroll=ku, wpc=wpc, pad=pad)
            c.pop("current", None)
            if all(c != {k: v for k, v in d.items() if k != "current"} for d in cs):
                cs.append(c)
        out[n] = cs
    print(json.dumps(out))


if __name__ == "__main__":
    main()
