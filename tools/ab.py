#!/usr/bin/env python3
"""A/B a tuning knob on the GPU box: rebuild with each define set, sweep, tag.

    python tools/ab.py --variant base="JM_DMMA_KCOMPACT=0 JM_DMMA_BORDER_MAX=2" --variant new= \
        --sizes 17,18,19,20 --dtypes f64 --repeats 100 --out gpurun_out/ab.jsonl

Each variant sets JM_BUILD_DEFINES (jm_plan.h knobs, applied identically to
the host planner, the AoT cubin and the NVRTC source: _build.py), force-
rebuilds libjitmat.so in the box's scratch copy, and runs tools/stream_sweep.py;
every JSON line gets {"ab": name, "defines": ...}.  The last variant's build is
left in place, so list the default last.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def table(path: str) -> None:
    """rows (n, dtype, R) x columns (variant): the library's own pick ("auto"),
    fraction of HBM for R(n+1) < 46 else of the FP pipe"""
    rows, names = {}, []
    for ln in open(path):
        d = json.loads(ln)
        if d["ab"] not in names:
            names.append(d["ab"])
        hbm = d["repeat"] * (d["n"] + 1) < 46
        f = d["auto"]["frac_hbm" if hbm else "frac_pipe"]
        rows.setdefault((d["dtype"], d["repeat"], d["n"]), {})[d["ab"]] = (f, d["kernels"]["0"]["regs"])
    print("| dtype | R | n | " + " | ".join(names) + " |")
    print("|---|---|---|" + "---|" * len(names))
    for k in sorted(rows):
        cells = [f"{rows[k][v][0]:.3f} ({rows[k][v][1]} r)" if v in rows[k] else "-" for v in names]
        print(f"| {k[0]} | {k[1]} | {k[2]} | " + " | ".join(cells) + " |")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--variant", action="append", help='name="DEF=V DEF2=V2"')
    ap.add_argument("--table", default=None, help="print a JSONL file of this tool as a table and exit")
    ap.add_argument("--sizes", default="")
    ap.add_argument("--dtypes", default="f64")
    ap.add_argument("--repeats", default="100")
    ap.add_argument("--gb", type=float, default=0.5)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--tool", default="stream_sweep", choices=["stream_sweep", "mass_bench"],
                    help="mass_bench: the Laghos mass action (tools/mass_bench.py) instead of the update sweep")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    if a.table:
        table(a.table)
        return
    sizes = []
    for part in filter(None, a.sizes.split(",")):
        lo, _, hi = part.partition("..")
        sizes += list(range(int(lo), int(hi or lo) + 1))
    for v in a.variant:
        name, _, defs = v.partition("=")
        env = dict(os.environ, JM_BUILD_DEFINES=defs.strip('"'))
        b = subprocess.run([sys.executable, "-c", "import paper_1904_08555_b200._build as b; b.build(force=True)"],
                           cwd=ROOT, env=env, capture_output=True, text=True)
        if b.returncode:
            print(f"{name}: build failed: {b.stderr[-2000:]}", file=sys.stderr)
            continue
        cmd = ([os.path.join(ROOT, "tools", "mass_bench.py"), "--pairs", "all", "--elements", "2097152"]
               if a.tool == "mass_bench" else
               [os.path.join(ROOT, "tools", "stream_sweep.py"), "--sizes", ",".join(map(str, sizes)),
                "--dtypes", a.dtypes, "--repeats", a.repeats, "--gb", str(a.gb), "--steps", str(a.steps)])
        p = subprocess.run([sys.executable] + cmd, cwd=ROOT, env=env, capture_output=True, text=True)
        if p.returncode:
            print(f"{name}: sweep failed: {p.stderr[-2000:]}", file=sys.stderr)
        with open(a.out, "a") as fh:
            for ln in p.stdout.splitlines():
                d = json.loads(ln)
                d["ab"] = name
                d["defines"] = defs
                fh.write(json.dumps(d) + "\n")
        print(f"{name} done", file=sys.stderr, flush=True)


if __name__ == "__main__":
    main()
