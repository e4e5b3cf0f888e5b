#!/usr/bin/env python3
"""Render a tools/sweep.py JSON-lines file as a markdown report.

    python tools/make_report.py profiles/r01_sweep_final.jsonl > profiles/r01_sweep.md
"""
from __future__ import annotations

import json
import sys


def main(path: str) -> None:
    rows = [json.loads(ln) for ln in open(path) if ln.strip()]
    print(f"# Configuration sweep — `{path}` (tools/sweep.py, one B200)\n")
    import os
    hbm = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                      "MEASURED_PEAKS.json")))["hbm_gbs"]
    print(f"Roofline denominators: HBM {hbm} GB/s (MEASURED_PEAKS.json); FP64 37.2 TF and FP32 74.4 TF "
          "(148 SM x 64 / 128 FMA/clk x 2 x 1.965 GHz, DESIGN.md §6). Batch = 8 GB of input per config, "
          "`bench` inputs; generic = the AoT runtime-N kernel on the same inputs.\n")
    c3 = [d for d in rows if d["config"] == "C3"]
    if c3:
        print("## C3 — N sweep\n")
        print("| n | dtype | R | tile | variant | regs | spec ms | spec TF | frac HBM | frac pipe | generic ms | spec/generic |")
        print("|---|---|---|---|---|---|---|---|---|---|---|---|")
        for d in c3:
            s, g = d["specialized"], d["generic"]
            print(f"| {d['n']} | {d['dtype']} | {d['repeat']} | {d['tile']} | {d.get('variant', 'resident')} | "
                  f"{d['regs']} | {s['ms']:.2f} | "
                  f"{s['tflops']:.2f} | {s['frac_hbm']:.3f} | {s['frac_pipe']:.3f} | {g['ms']:.2f} | {d['speedup']:.2f} |")
    for d in rows:
        if d["config"] == "C1":
            print(f"\n## C1\n\nn=4 FP64 paper init, repeat 1000, one matrix: first call incl. NVRTC "
                  f"{d['first_call_ms_incl_nvrtc']:.1f} ms; warm launch {d['warm_launch_us_median']:.1f} us; "
                  f"result vs closed-form fixed point a*(4) = 1.0002501125631647: "
                  f"{d['max_ulps_from_fixed_point']:.0f} ulp.")
    c4 = [d for d in rows if d["config"] == "C4"]
    if c4:
        print("\n## C4 — mixed N (2^18 matrices, n ~ U{2..64}, repeat 10)\n")
        for d in c4:
            w = d["warm"]
            print(f"* {d['dtype']}: {d['compilations']} NVRTC compiles; cold pass one key at a time "
                  f"{d['cold_pass_s_incl_compiles']:.2f} s (median {d['compile_ms_per_key_median']:.0f} ms/key, "
                  f"max {d['compile_ms_per_key_max']:.0f}); cold pass via jit_mat_run_many (parallel compiles) "
                  f"{d['cold_pass_s_run_many_parallel_compiles']:.2f} s; warm run_many "
                  f"{w['specialized']['tflops']:.1f} TF ({w['specialized']['ms']:.2f} ms), serial per-group "
                  f"{w['specialized_serial']['tflops']:.1f} TF, generic {w['generic']['tflops']:.1f} TF "
                  f"(specialized/generic {d['specialized_speedup']:.2f}x)")


if __name__ == "__main__":
    main(sys.argv[1])
