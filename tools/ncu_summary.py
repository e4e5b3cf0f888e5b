#!/usr/bin/env python3
"""Summarise `ncu --set full` captures of the update kernels -> markdown rows / JSON.

    python tools/ncu_summary.py REP.ncu-rep [...] [--algo n,dtype,batch,repeat ...] [--json]

For each report (one captured launch of a `k_update*` kernel) it reads the raw
page in base units and prints the numbers the roofline argument needs
(DESIGN.md §6, §7): duration and SM clock, registers / shared memory /
warps active, the pipe the kind is bound by (FP64 "shared" pipe = DFMA +
DMMA, FMA pipe for FP32), DRAM bytes read + written against the algorithmic
2·n²·s·batch, shared-memory wavefronts and bank conflicts, and the top stall
reasons.  `--algo` gives the configuration of each report (same order) so the
algorithmic bytes and flops can be put beside the measured ones.
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import subprocess

STALLS = ["wait", "math_pipe_throttle", "short_scoreboard", "long_scoreboard", "mio_throttle", "barrier",
          "not_selected", "dispatch_stall", "lg_throttle", "branch_resolving", "no_instructions", "membar",
          "drain", "sleeping", "tex_throttle", "imc_miss", "misc"]


def raw(rep: str) -> list[dict]:
    """rows of the raw page: from a report (ncu -i) or a saved raw CSV (.csv / .csv.gz)"""
    if rep.endswith(".csv") or rep.endswith(".csv.gz"):
        import gzip
        out = gzip.open(rep, "rt").read() if rep.endswith(".gz") else open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-units", "base"],
                             check=True, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units = rows[0], rows[1]
    recs = [dict(zip(head, r)) for r in rows[2:]]
    # a saved page without --print-units base: scale to base units (ns, byte, Hz)
    scale = {"us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "s": 1e9, "second": 1e9,
             "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Kbyte/block": 1e3, "Mbyte/block": 1e6,
             "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9, "Kbyte/second": 1e3, "Mbyte/second": 1e6, "Gbyte/second": 1e9}
    for k, u in zip(head, units):
        f = scale.get(u)
        if f:
            for d in recs:
                try:
                    d[k] = str(float(d[k].replace(",", "")) * f)
                except (ValueError, KeyError):
                    pass
    return recs


def num(d: dict, k: str) -> float:
    v = d.get(k, "")
    try:
        return float(str(v).replace(",", ""))
    except ValueError:
        return float("nan")


def summarise(d: dict, algo=None) -> dict:
    s = {
        "kernel": d.get("Kernel Name", "?"),
        "grid": d.get("Grid Size"), "block": d.get("Block Size"),
        "ms": num(d, "gpu__time_duration.sum") / 1e6,
        "sm_ghz": num(d, "sm__cycles_elapsed.avg.per_second") / 1e9,
        "regs": int(num(d, "launch__registers_per_thread")),
        "smem_kb": num(d, "launch__shared_mem_per_block_dynamic") / 1e3,
        "occ_limit_regs": num(d, "launch__occupancy_limit_registers"),
        "occ_limit_smem": num(d, "launch__occupancy_limit_shared_mem"),
        "warps_active_pct": num(d, "sm__warps_active.avg.pct_of_peak_sustained_active"),
        "fp64_shared_pipe_pct": num(d, "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active"),
        "dmma_pct": num(d, "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active"),
        "dfma_pct": num(d, "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
        "fma_pipe_pct": num(d, "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
        "issue_active_pct": num(d, "sm__inst_executed.avg.pct_of_peak_sustained_active"),
        "dram_read": num(d, "dram__bytes_read.sum"),
        "dram_write": num(d, "dram__bytes_write.sum"),
        "dram_pct": num(d, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
        "smem_wavefronts": num(d, "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
        "smem_conflicts": num(d, "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
        # wavefronts above the ideal for the accessed addresses (the source page's
        # "L1 Wavefronts Shared Excessive"); the bank-conflict counter above also
        # counts the extra wavefronts every 128-bit access needs, so it is not
        # the excess
        "smem_excessive": num(d, "derived__memory_l1_wavefronts_shared_excessive"),
        "smem_pipe_pct": num(d, "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
        "inst": num(d, "smsp__inst_executed.sum"),
    }
    st = {}
    for k in STALLS:
        v = num(d, f"smsp__average_warps_issue_stalled_{k}_per_issue_active.ratio")
        if v == v and v > 0.02:
            st[k] = round(v, 2)
    s["stalls_per_issue"] = dict(sorted(st.items(), key=lambda kv: -kv[1])[:5])
    if algo:
        n, dt, batch, rep = algo
        es = 8 if dt == "f64" else 4
        s["algo_bytes"] = 2 * n * n * es * batch
        s["algo_flops"] = batch * rep * (2 * n ** 3 + 2 * n * n)
        s["traffic_ratio"] = (s["dram_read"] + s["dram_write"]) / s["algo_bytes"]
        s["achieved_tflops"] = s["algo_flops"] / (s["ms"] * 1e-3) / 1e12
        s["achieved_gbs"] = s["algo_bytes"] / (s["ms"] * 1e-3) / 1e9
    return s


def md_row(s: dict) -> str:
    pipe = (f"shared {s['fp64_shared_pipe_pct']:.1f}% (dmma {s['dmma_pct']:.1f}, dfma {s['dfma_pct']:.1f})"
            if s["fp64_shared_pipe_pct"] > 1 else f"fma {s['fma_pipe_pct']:.1f}%")
    tr = f"{s['traffic_ratio']:.3f}" if "traffic_ratio" in s else "-"
    conf = s["smem_excessive"] / s["smem_wavefronts"] if s["smem_wavefronts"] > 0 else 0.0
    return (f"| {s['kernel'].split('(')[0]} | {s['ms']:.3f} | {s['regs']} | {s['smem_kb']:.1f} | "
            f"{s['warps_active_pct']:.1f} | {pipe} | {s['dram_pct']:.1f} | {tr} | "
            f"{s['smem_wavefronts'] / 1e6:.1f}M ({100 * conf:.0f}% excess) | "
            f"{', '.join(f'{k} {v}' for k, v in s['stalls_per_issue'].items())} |")


HEADER = ("| kernel | ms | regs | smem KB | warps active % | pipe busy | DRAM % peak | DRAM/algo bytes | "
          "smem wavefronts | top stalls (per issue) |\n|---|---|---|---|---|---|---|---|---|---|")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("reps", nargs="+")
    ap.add_argument("--algo", nargs="*", default=[], help="n,dtype,batch,repeat per captured launch, in order")
    ap.add_argument("--json", action="store_true")
    a = ap.parse_args()
    algos = []
    for x in a.algo:
        n, dt, b, r = x.split(",")
        algos.append((int(n), dt, int(b), int(r)))
    if not a.json:
        print(HEADER)
    i = 0   # --algo entries apply to the captured update launches in order, across reports
    for rep in a.reps:
        for d in raw(rep):
            if not any(k in d.get("Kernel Name", "") for k in ("k_update", "k_matmul", "k_mass", "jm_generic")):
                continue
            s = summarise(d, algos[i] if i < len(algos) else None)
            i += 1
            s["report"] = rep
            print(json.dumps(s) if a.json else md_row(s))


if __name__ == "__main__":
    main()
