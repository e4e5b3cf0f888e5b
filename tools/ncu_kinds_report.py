#!/usr/bin/env python3
"""Render the per-kind ncu capture (tools/ncu_kinds.py configs, summarised by
tools/ncu_summary.py --json) as the markdown table under profiles/.

    python tools/ncu_kinds_report.py profiles/r02_ncu_kinds.jsonl > profiles/r02_ncu_kinds.md

Per launch: the kind, the configuration, the roofline side it sits on
(HBM when R(n+1) < 46, else the FP64 / FP32 pipe: DESIGN.md §6), the
achieved fraction of that roof from ncu's own duration (serialised,
cold-cache replay, so slightly below the bench numbers), the pipe the kind
issues to, DRAM bytes against the algorithmic 2·n²·s·batch, shared-memory
shared-memory wavefronts above the ideal for the addresses accessed (ncu's
"excessive" wavefronts; the raw bank-conflict counter also counts the
second wavefront every 128-bit access needs, so it overstates conflicts),
occupancy and the top stall reasons.
"""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))

import ncu_kinds  # noqa: E402

HBM = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
PEAK = {"f64": 148 * 64 * 2 * 1.965e9 / 1e12, "f32": 148 * 128 * 2 * 1.965e9 / 1e12}


def main(path: str) -> None:
    rows = [json.loads(ln) for ln in open(path) if ln.strip()]
    print(f"# Per-kind ncu capture — `{os.path.basename(path)}` (one B200, `ncu --set full --clock-control none`)\n")
    print("One launch of every tiling kind the planner ships (`tools/ncu_kinds.py`, inputs ~0.5 GB > L2), "
          "summarised by `tools/ncu_summary.py`. Roof: HBM "
          f"{HBM:.0f} GB/s (MEASURED_PEAKS.json) when R(n+1) < 46, else the FP64 37.2 / FP32 74.4 TF pipe "
          "(DESIGN.md §6). ncu replays each kernel serialised and cold, so its fractions run a little under "
          "the bench / sweep numbers. DRAM/algo = (dram read + write) / (2·n²·s·batch).\n")
    print("| kind | config | roof | achieved | frac | pipe busy | DRAM/algo | regs | smem KB | warps active % | "
          "smem excess wavefronts | top stalls |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|")
    for (what, n, dt, r, v), s in zip(ncu_kinds.KINDS, rows):
        hbm = r * (n + 1) < 46
        if hbm:
            ach, frac, roof = s["achieved_gbs"], s["achieved_gbs"] / HBM, "HBM"
            ach_s = f"{ach:.0f} GB/s"
        else:
            ach, frac, roof = s["achieved_tflops"], s["achieved_tflops"] / PEAK[dt], f"{dt.upper()} pipe"
            ach_s = f"{ach:.2f} TF"
        pipe = (f"FP64 {s['fp64_shared_pipe_pct']:.0f}% (DMMA {s['dmma_pct']:.0f}, DFMA {s['dfma_pct']:.0f})"
                if dt == "f64" else f"FMA {s['fma_pipe_pct']:.0f}%")
        conf = s.get("smem_excessive", float("nan")) / s["smem_wavefronts"] if s["smem_wavefronts"] > 0 else 0.0
        st = ", ".join(f"{k} {v}" for k, v in list(s["stalls_per_issue"].items())[:3])
        name = s["kernel"].replace("void ", "").split("(")[0]
        print(f"| {what} (`{name}`) | n={n} {dt} R={r} batch={s['algo_bytes'] // (2 * n * n * (8 if dt == 'f64' else 4))} "
              f"| {roof} | {ach_s} | {frac:.2f} | {pipe} | {s['traffic_ratio']:.3f} | {s['regs']} | "
              f"{s['smem_kb']:.1f} | {s['warps_active_pct']:.0f} | {100 * conf:.0f}% | {st} |")


if __name__ == "__main__":
    main(sys.argv[1])
