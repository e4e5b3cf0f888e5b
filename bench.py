#!/usr/bin/env python3
"""bench.py — throughput of the JIT-specialized batched Eigen-benchmark update.

Headline workload (BASELINE.json configs[1], "C2"): a batch of 2^20 FP64 16x16
matrices per GPU, each updated M <- Ones + 5e-5 (M + M*M) 100 times
(Listings 4/5), by the NVRTC-specialized kernel; the generic
runtime-N kernel is timed beside it on the same inputs.  One "step" is one
jit_mat_run over the whole batch (every row of SURVEY.md §8(a): key lookup,
load, 100 updates, store).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
    torchrun --nproc-per-node N bench.py --gpus N ...        (N > 1)

Rank 0 prints ONE JSON line.  Multi-GPU: each rank owns its own slice of the
global batch (global matrix index rank*batch + b, so inputs are W-invariant),
no data-path collective; NCCL only gathers the per-rank timing/checksum record
after the timed region.  value = all ranks' matrix-updates
/ max-over-ranks device time.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

with open(os.path.join(ROOT, "BASELINE.json")) as _f:
    METRIC = json.load(_f)["metric"]
UNIT = "matrix-updates/s"
NOMINAL_FP64_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12   # 37.2 TF
NOMINAL_FP32_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12  # 74.4 TF


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=None,
                    help="GPUs (one rank each); N > 1 without torchrun re-launches itself under "
                         "torch.distributed.run (default: WORLD_SIZE, else 1)")
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    # (--size: the same option under torchrun, whose own parser takes --n for --nnodes)
    ap.add_argument("--n", "--size", dest="n", type=int, default=16)
    ap.add_argument("--dtype", default="f64", choices=["f64", "f32"])
    ap.add_argument("--batch", type=int, default=1 << 20, help="matrices per GPU")
    ap.add_argument("--global-batch", type=int, default=None,
                    help="strong scaling (configs[4], C5): fixed total batch split across ranks")
    ap.add_argument("--repeat", type=int, default=100)
    ap.add_argument("--addend", default="ones", choices=["ones", "identity"])
    ap.add_argument("--kind", default="specialized", choices=["specialized", "generic"])
    ap.add_argument("--no-generic", action="store_true", help="skip the generic side-by-side")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true", help="skip the oracle cpu_baseline")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--out", default=None, help="also append the JSON line to this file")
    return ap.parse_args()


def flops_per_update(n: int, addend: str) -> int:
    # 2n^3 - n^2 for M*M, + n^2 (M + .), + n^2 (c * .), + n^2 (A + .) = 2n^3 + 2n^2;
    # Identity adds only the n diagonal ones.
    return 2 * n ** 3 + 2 * n * n if addend == "ones" else 2 * n ** 3 + n * n + n


def workload_name(a) -> str:
    tag = "C2" if (a.n, a.dtype, a.batch, a.repeat) == (16, "f64", 1 << 20, 100) else "custom"
    return (f"{tag}: batch {a.batch} x {a.dtype.upper()} {a.n}x{a.n} per GPU, repeat {a.repeat}, "
            f"addend {a.addend}, {a.kind} kernel")


# ------------------------------------------------------------------ clocks
_REASONS = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]


class ClockSampler:
    """nvidia-smi at 200 ms during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index: int):
        q = ("clocks.sm,clocks.max.sm,power.draw,utilization.gpu,"
             + ",".join(f"clocks_event_reasons.{r}" for r in _REASONS))
        self.cmd = ["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                    "-lms", "200", "-i", str(index)]
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(self.cmd, stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                                         text=True)
        except OSError:
            self.proc = None
        time.sleep(0.25)
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [ln for ln in out.splitlines() if ln.strip()]
        return False

    def summary(self) -> dict:
        rows = []
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 4 + len(_REASONS):
                continue
            try:
                rows.append({"sm": float(f[0]), "max": float(f[1]), "power": float(f[2]),
                             "util": float(f[3]),
                             "reasons": [r for r, v in zip(_REASONS, f[4:]) if v.lower() == "active"]})
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        load = [r for r in rows if r["util"] >= 50] or rows
        reasons = sorted({x for r in load for x in r["reasons"]})
        return {"sm_mhz": statistics.median(r["sm"] for r in load),
                "sm_max_mhz": max(r["max"] for r in rows), "reasons": reasons,
                "samples": len(rows), "samples_under_load": len(load),
                "power_w_max": max(r["power"] for r in rows)}


# ------------------------------------------------------------------ oracle leg
def time_oracle(a, seconds: float) -> dict:
    """Time the CPU oracle (as it stands) on a bounded sample of the same workload."""
    import numpy as np

    import jm_synth
    import oracle

    threads = oracle.default_threads()
    seed = jm_synth.SEED_BENCH
    pilot = threads * 4
    while True:   # pilot until it takes >= 0.3 s, so the rate estimate is not start-up bound
        x = jm_synth.generate(a.n, a.dtype, "bench", seed, 0, pilot)
        t0 = time.perf_counter()
        oracle.run(x, a.repeat, a.addend, threads=threads)
        dt = max(time.perf_counter() - t0, 1e-6)
        if dt >= 0.3 or pilot >= a.batch:
            break
        pilot = min(a.batch, pilot * max(2, int(0.4 / dt)))
    per_matrix = dt / pilot
    sample = int(min(a.batch, max(threads, seconds / per_matrix)))
    x = jm_synth.generate_chunked(a.n, a.dtype, "bench", seed, 0, sample)
    t0 = time.perf_counter()
    oracle.run(x, a.repeat, a.addend, threads=threads)
    el = time.perf_counter() - t0
    ups = sample * a.repeat / el
    return {"value": ups, "unit": UNIT, "cores": threads, "kind": "oracle",
            "gflops": ups * flops_per_update(a.n, a.addend) / 1e9, "seconds": el,
            "sample": (f"first {sample} of the {a.batch} matrices of the same workload "
                       f"(n={a.n} {a.dtype} repeat={a.repeat}), plain C triple loop, "
                       f"{threads} threads; cpu {cpu_model()}")}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(a, rank: int) -> None:
    """--impl reference: the oracle is this tier's reference arm (rank 0 only)."""
    if rank != 0:
        return
    import jm_synth
    import oracle

    threads = oracle.default_threads()
    total_budget = 150.0
    per_step = min(2.0, total_budget / max(1, a.steps + a.warmup))
    cal = time_oracle(a, max(0.5, per_step))
    sample = int(min(a.batch, max(threads, cal["value"] * per_step / a.repeat)))
    x = jm_synth.generate_chunked(a.n, a.dtype, "bench", jm_synth.SEED_BENCH, 0, sample)
    for _ in range(a.warmup):
        oracle.run(x, a.repeat, a.addend, threads=threads)
    times = []
    for _ in range(a.steps):
        t0 = time.perf_counter()
        oracle.run(x, a.repeat, a.addend, threads=threads)
        times.append(time.perf_counter() - t0)
    ms = 1e3 * sum(times) / len(times)
    value = sample * a.repeat / (ms / 1e3)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": a.gpus, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": a.dtype, "data": "synthetic", "impl": "reference",
        "config": {"workload": workload_name(a), "n": a.n, "repeat": a.repeat,
                   "batch_per_step": sample, "dist": "bench U[-1,1)"},
        "gflops": value * flops_per_update(a.n, a.addend) / 1e9,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle",
                         "sample": (f"each step: first {sample} matrices of the workload, "
                                    f"{threads} host threads; cpu {cpu_model()}")},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line, a)


def emit(line: dict, a) -> None:
    s = json.dumps(line)
    print(s, flush=True)
    if a.out:
        with open(a.out, "a") as f:
            f.write(s + "\n")


def free_port() -> int:
    import socket
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch(a) -> int:
    """`bench.py --gpus N` (N > 1) started as a plain process: run the same
    command as N ranks under torch.distributed.run (one process per GPU,
    rendezvous on 127.0.0.1), so the driver's command line and torchrun's
    give the same job."""
    # torch.distributed.run's own parser takes "--n" as an abbreviation of its
    # --nnodes / --nproc-per-node even after the script: pass it as --size
    args = ["--size" + x[3:] if x == "--n" or x.startswith("--n=") else x for x in sys.argv[1:]]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}",
           os.path.abspath(__file__), *args]
    return subprocess.call(cmd)


def resolve_world(a) -> tuple[int, int, int]:
    """(world, rank, local_rank) from the torchrun environment, checked against --gpus."""
    env_world = os.environ.get("WORLD_SIZE")
    world = int(env_world) if env_world is not None else 1
    if a.gpus is None:
        a.gpus = world
    if env_world is not None and world != a.gpus:
        raise SystemExit(f"bench.py: --gpus {a.gpus} but WORLD_SIZE={world}: launch one rank per GPU")
    return world, int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0"))


# ------------------------------------------------------------------ GPU leg
def main():
    a = parse()
    if a.impl != "reference" and (a.gpus or 1) > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(a))
    world, rank, local = resolve_world(a)
    if os.environ.get("JM_BENCH_DRY_RUN"):    # test hook: the launch contract only, no GPU work
        # one write(2) per record: the ranks share the pipe, and print() may split a line
        os.write(1, (json.dumps({"rank": rank, "world": world, "gpus": a.gpus, "local_rank": local}) + "\n").encode())
        return
    if a.impl == "reference":     # (rank 0 only; n_gpus = --gpus, as in the GPU arm)
        run_reference(a, rank)
        return

    import torch
    import torch.distributed as dist

    import paper_1904_08555_b200 as jm
    from paper_1904_08555_b200 import shard

    # one process per GPU over NCCL; JM_BENCH_DIST_BACKEND=gloo (test hook)
    # runs the same N > 1 path with ranks sharing the visible GPUs and the
    # record gather on CPU, so the multi-rank logic can be exercised on a 1-GPU box
    backend = os.environ.get("JM_BENCH_DIST_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    cdev = dev if backend == "nccl" else torch.device("cpu")    # collective tensors
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    torch.cuda.init()
    jm.jit_mat_init(local)
    stream = torch.cuda.Stream(device=dev)
    jm.jit_mat_set_stream(stream.cuda_stream)

    n, dt, R = a.n, a.dtype, a.repeat
    tdt = torch.float64 if dt == "f64" else torch.float32
    es = 8 if dt == "f64" else 4
    if a.global_batch is not None:     # strong scaling: every N shares one fixed global batch
        gfirst, B = shard.strong_slice(rank, world, a.global_batch)
        a.batch = B
    else:                              # weak scaling: B matrices per GPU
        B = a.batch
        gfirst, _ = shard.weak_slice(rank, B)
    x = torch.empty(B, n, n, dtype=tdt, device=dev)
    y = torch.empty_like(x)

    def barrier():
        if world > 1:
            if backend == "nccl":
                dist.barrier(device_ids=[local])
            else:
                dist.barrier()

    with torch.cuda.stream(stream):
        jm.jit_mat_fill(n, dt, 1, 0x0019040855, gfirst, B, x.data_ptr())
    stream.synchronize()

    # ---- multi-GPU: rank 0 specializes, the others import its cubins over
    # NCCL instead of running NVRTC themselves
    # ---- first call: NVRTC specialization (reported separately, never timed);
    # under N > 1 it is rank 0's compile, which the other ranks then import
    first_call_ms = None
    if world > 1 and a.kind == "specialized":
        blob = None
        if rank == 0:
            t0 = time.perf_counter()
            jm.jit_mat_prepare_for(n, dt, R, a.addend, a.kind)
            first_call_ms = (time.perf_counter() - t0) * 1e3
            blob = jm.jit_mat_cache_export(n, dt, a.addend)
        blob = shard.broadcast_blob(dist, blob, 0, cdev)
        if rank != 0:
            jm.jit_mat_cache_import(blob)

    t0 = time.perf_counter()
    # the kernel this repeat count selects: resident, or the streaming variant
    # on the HBM-bound side (include/jit_mat.h VARIANT)
    variant = jm.jit_mat_prepare_for(n, dt, R, a.addend, a.kind)
    if first_call_ms is None:
        first_call_ms = (time.perf_counter() - t0) * 1e3
    key = [k for k in jm.jit_mat_key_info()
           if k["op"] == 0 and k["n"] == n and k["dtype"] == (1 if dt == "f64" else 0)
           and k["kind"] == {"specialized": 0, "generic": 1, "aot_specialized": 2}[a.kind]
           and k["addend"] == (0 if a.addend == "ones" else 1) and k["variant"] == variant][0]

    def step(kind):
        jm.jit_mat_run_ex(n, dt, B, R, x.data_ptr(), y.data_ptr(), addend=a.addend, kind=kind,
                          stream=stream.cuda_stream)

    def timed(kind, steps, warmup):
        for _ in range(warmup):
            step(kind)
        stream.synchronize()
        barrier()
        torch.cuda.synchronize()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        l0 = jm.jit_mat_stats()["launches"]
        ev0.record(stream)
        for _ in range(steps):
            step(kind)
        ev1.record(stream)
        ev1.synchronize()
        launches = jm.jit_mat_stats()["launches"] - l0
        barrier()
        torch.cuda.synchronize()
        return ev0.elapsed_time(ev1), launches

    with ClockSampler(local) as clk:
        el_ms, launches = timed(a.kind, a.steps, max(3, a.warmup))
    clocks = clk.summary()
    ms_step = el_ms / a.steps

    # max over ranks + checksum gather (NCCL, outside the data path)
    csum, _ = jm.jit_mat_checksum(n, dt, gfirst, B, y.data_ptr())
    if world > 1:
        recs, cks = shard.gather_record(dist, [ms_step, float(B)], [csum], cdev)
    else:
        recs, cks = [[ms_step, float(B)]], [[csum]]
    ms_max = max(r[0] for r in recs)
    total_units = sum(r[1] for r in recs) * R
    value = total_units / (ms_max / 1e3)
    global_checksum = shard.combine_checksums(c[0] for c in cks)

    fpu = flops_per_update(n, a.addend)
    # the dominant kernel's rate per GPU: the largest slice over the slowest
    # rank's launch time (max over ranks, as `value`)
    b_max = max(r[1] for r in recs)
    achieved_tf = b_max * R * fpu / (ms_max / 1e3) / 1e12
    peak_tf = NOMINAL_FP64_TFLOPS if dt == "f64" else NOMINAL_FP32_TFLOPS
    alg_bytes = 2 * int(b_max) * n * n * es
    hbm_gbs = alg_bytes / (ms_max / 1e3) / 1e9
    # which roofline binds: compare ideal compute vs ideal HBM time
    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
        peaks = json.load(f)
    t_comp = b_max * R * fpu / (peak_tf * 1e12)
    t_hbm = alg_bytes / (peaks["hbm_gbs"] * 1e9)
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            traffic = json.load(f).get(f"{n}/{dt}/{B}/{R}/{a.kind}")
    if t_comp >= t_hbm:
        roof = {"bound": "alu", "pipe": "fp64 (DMMA.8x8x4 + DFMA share it)" if dt == "f64"
                else "fp32 (FFMA2)",
                "achieved": achieved_tf, "peak": peak_tf, "unit": "TFLOP/s",
                "frac": achieved_tf / peak_tf, "traffic": traffic,
                "peak_source": ("derived: 148 SM x %d FMA/clk x 2 x 1.965 GHz (DESIGN.md); "
                                "microbench measured DMMA 36.95 / DFMA 36.74 TF (profiles/r01_microbench_peaks.json)"
                                % (64 if dt == "f64" else 128)),
                "algorithmic_flops_per_launch": int(b_max) * R * fpu,
                "hbm_gbs_achieved": hbm_gbs}
        # the same fraction against this pool's measured pipe peak (SURVEY.md §7
        # hard part 3: nominal and measured side by side)
        mb = os.path.join(ROOT, "profiles", "r01_microbench_peaks.json")
        if os.path.exists(mb):
            with open(mb) as f:
                mpk = json.load(f).get("dmma_tflops" if dt == "f64" else "ffma2_tflops")
            if mpk:
                roof["peak_measured"] = mpk
                roof["frac_of_measured"] = achieved_tf / mpk
    else:
        roof = {"bound": "hbm", "achieved": hbm_gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": hbm_gbs / peaks["hbm_gbs"], "traffic": traffic,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs",
                "algorithmic_bytes_per_launch": alg_bytes, "tflops_achieved": achieved_tf}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": a.gpus, "steps": a.steps,
        "warmup": max(3, a.warmup), "ms_per_step": ms_max, "higher_is_better": True,
        "scaling": "strong" if a.global_batch is not None else "weak",
        "vs_baseline": None, "dtype": dt, "data": "synthetic",
        "config": {"workload": workload_name(a), "n": n, "batch_per_gpu": B,
                   "global_batch": a.global_batch if a.global_batch is not None else B * world,
                   "repeat": R, "addend": a.addend, "kind": a.kind,
                   "dist": "bench: U[-1,1) counter-hash, seed 0x0019040855",
                   "l2": f"inputs {alg_bytes / 2 / 1e9:.2f} GB per GPU > 126 MB L2 (no flush needed)",
                   "parallelism": f"dp{world} (contiguous batch slices, no data-path collective)"},
        "gflops": value * fpu / 1e9,
        "roofline": roof,
        "clocks": clocks,
        "gpu_launches": launches,
        "nvrtc_first_call_ms": first_call_ms,
        "specializations": (f"rank 0 compiled, ranks 1..N-1 imported its cubins ({backend} broadcast)"
                            if world > 1 and a.kind == "specialized" else "compiled in this process"),
        "collective_backend": backend if world > 1 else None,
        "kernel": {"tile": key["tile_name"], "variant": "streaming" if variant else "resident",
                   "regs": key["regs"], "local_bytes": key["local_bytes"],
                   "smem_bytes": key["smem_bytes"], "threads": key["threads"],
                   "compile_ms": key["compile_ms"], "cubin_bytes": key["cubin_bytes"]},
        "checksum_u64": f"{global_checksum:016x}",
    }

    # ---- generic runtime-N kernel, same inputs (the un-specialized comparison)
    if not a.no_generic and a.kind == "specialized":
        gsteps = max(2, min(5, a.steps))
        g_ms, _ = timed("generic", gsteps, 1)
        g_ms_step = g_ms / gsteps
        g_max = (max(r[0] for r in shard.gather_record(dist, [g_ms_step], [], cdev)[0])
                 if world > 1 else g_ms_step)
        gval = total_units / (g_max / 1e3)
        line["generic"] = {"value": gval, "unit": UNIT, "ms_per_step": g_max,
                           "gflops": gval * fpu / 1e9,
                           "specialized_speedup": value / gval}
        # Fig. 3's third bar: the same template compiled ahead of time (n = 3, 7, 16 double)
        if dt == "f64" and n in (3, 7, 16):
            a_ms, _ = timed("aot_specialized", gsteps, 1)
            a_max = (max(r[0] for r in shard.gather_record(dist, [a_ms / gsteps], [], cdev)[0])
                     if world > 1 else a_ms / gsteps)
            aval = total_units / (a_max / 1e3)
            line["aot_specialized"] = {"value": aval, "unit": UNIT, "ms_per_step": a_max,
                                       "time_relative_to_jit": a_max / ms_max}

    # ---- end to end through the public C ABI with HOST buffers
    if not a.no_e2e:
        e2e_steps = max(2, min(5, a.steps))
        hx = torch.empty(B, n, n, dtype=tdt, pin_memory=True)
        hy = torch.empty(B, n, n, dtype=tdt, pin_memory=True)
        hx.copy_(x.cpu())
        jm.jit_mat_run_host(n, dt, B, R, hx.data_ptr(), hy.data_ptr())   # warm-up
        barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            jm.jit_mat_run_host(n, dt, B, R, hx.data_ptr(), hy.data_ptr())
        el = time.perf_counter() - t0
        e_max = (max(r[0] for r in shard.gather_record(dist, [el / e2e_steps], [], cdev)[0])
                 if world > 1 else el / e2e_steps)
        line["e2e"] = {"value": total_units / e_max, "unit": UNIT,
                       "h2d_bytes_per_step": B * n * n * es, "d2h_bytes_per_step": B * n * n * es,
                       "ms_per_step": e_max * 1e3, "steps": e2e_steps,
                       "api": "jit_mat_run_host (pinned host in/out, chunked H2D/compute/D2H overlap)"}
        del hx, hy

    if rank == 0 and world == 1 and not a.no_cpu:
        line["cpu_baseline"] = time_oracle(a, a.cpu_seconds)
        line["cpu_baseline"]["value_vs_gpu"] = value / line["cpu_baseline"]["value"]

    if rank == 0:
        emit(line, a)
    if world > 1:
        barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
