#!/usr/bin/env python3
"""Config sweep (BASELINE.json configs C1, C3, C4) on one B200 -> JSON lines.

    python tools/sweep.py [--only c1,c3,c4] [--out gpurun_out/sweep.jsonl]

C1  n=4 FP64 paper-init, batch 1, repeat 1000: first-call (NVRTC) latency,
    warm launch latency, result vs the closed-form fixed point.
C3  n in {2,3,4,8,16,32,64} x {f64,f32} x repeat in {1,100}, batch sized to
    8 GB of input, specialized and generic side by side; roofline fraction
    against HBM (measured 6458 GB/s) or the FP64/FP32 pipe (37.2 / 74.4 TF).
C4  2^18 matrices with n ~ U{2..64} (numpy PCG64(1904)), grouped by n, repeat
    10, FP64 then FP32: cold pass (every key compiles) then warm pass.
Not the bench contract line (bench.py is); this is the per-config report.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1904_08555_b200 as jm  # noqa: E402

HBM = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
PEAK = {"f64": 148 * 64 * 2 * 1.965e9 / 1e12, "f32": 148 * 128 * 2 * 1.965e9 / 1e12}
SEED = 0x0019040855


def fpu(n):
    return 2 * n ** 3 + 2 * n * n


def emit(d, fh):
    s = json.dumps(d)
    print(s, flush=True)
    if fh:
        fh.write(s + "\n")
        fh.flush()


def time_run(n, dt, B, R, x, y, kind, steps, warmup, stream):
    for _ in range(warmup):
        jm.jit_mat_run_ex(n, dt, B, R, x.data_ptr(), y.data_ptr(), kind=kind, stream=stream.cuda_stream)
    stream.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        jm.jit_mat_run_ex(n, dt, B, R, x.data_ptr(), y.data_ptr(), kind=kind, stream=stream.cuda_stream)
    e1.record(stream)
    e1.synchronize()
    return e0.elapsed_time(e1) / steps


def c1(fh, stream):
    n, R = 4, 1000
    x = torch.arange(16, dtype=torch.float64, device="cuda").reshape(1, 4, 4)  # iota = paper init
    y = torch.empty_like(x)
    t0 = time.perf_counter()
    jm.jit_mat_run_ex(n, "f64", 1, R, x.data_ptr(), y.data_ptr(), stream=stream.cuda_stream,
                      flags=jm.JM_FLAG_SYNC)
    first_ms = (time.perf_counter() - t0) * 1e3
    def warm_us(flags):
        v = []
        for _ in range(200):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            jm.jit_mat_run_ex(n, "f64", 1, R, x.data_ptr(), y.data_ptr(), stream=stream.cuda_stream, flags=flags)
            e1.record(stream)
            e1.synchronize()
            v.append(e0.elapsed_time(e1) * 1e3)
        return float(np.median(v))
    # the thread-per-matrix kernel (r01's C1 path) beside the latency kernel
    # the library now picks for a batch this small (a warp per matrix)
    jm.jit_mat_run_ex(n, "f64", 1, R, x.data_ptr(), y.data_ptr(), stream=stream.cuda_stream,
                      flags=jm.JM_FLAG_RESIDENT | jm.JM_FLAG_SYNC)
    tpm_us = warm_us(jm.JM_FLAG_RESIDENT)
    lat = [warm_us(0)]
    t0 = time.perf_counter()
    for _ in range(1000):
        jm.jit_mat_prepare(n, "f64")
    hit_ns = (time.perf_counter() - t0) / 1000 * 1e9
    out = y.cpu().numpy().ravel()
    emit({"config": "C1", "n": 4, "dtype": "f64", "batch": 1, "repeat": R,
          "first_call_ms_incl_nvrtc": first_ms, "warm_launch_us_median": float(np.median(lat)),
          "kernel": "latency (warp per matrix)", "thread_per_matrix_warm_us_median": tpm_us,
          "cache_hit_prepare_ns_python": hit_ns,
          "result": out.tolist(), "expected_fixed_point": 1.0002501125631647,
          "max_ulps_from_fixed_point": float(np.max(np.abs(out - 1.0002501125631647)) / 2.220446049250313e-16)},
         fh)


def c3(fh, stream, sizes, dtypes, repeats, steps):
    for dt in dtypes:
        es = 8 if dt == "f64" else 4
        tdt = torch.float64 if dt == "f64" else torch.float32
        for n in sizes:
            B = int(8e9 // (n * n * es))
            x = torch.empty(B, n, n, dtype=tdt, device="cuda")
            y = torch.empty_like(x)
            jm.jit_mat_fill(n, dt, 1, SEED, 0, B, x.data_ptr())
            torch.cuda.synchronize()
            for R in repeats:
                # the kernel this repeat count selects (resident or streaming variant)
                t0 = time.perf_counter()
                variant = jm.jit_mat_prepare_for(n, dt, R)
                comp = (time.perf_counter() - t0) * 1e3
                info = [k for k in jm.jit_mat_key_info() if k["op"] == 0 and k["n"] == n
                        and k["dtype"] == (1 if dt == "f64" else 0)
                        and k["kind"] == 0 and k["addend"] == 0 and k["variant"] == variant][0]
                row = {"config": "C3", "n": n, "dtype": dt, "batch": B, "repeat": R,
                       "tile": info["tile_name"], "variant": "streaming" if variant else "resident",
                       "regs": info["regs"], "smem": info["smem_bytes"],
                       "nvrtc_ms": info["compile_ms"], "first_prepare_ms": comp}
                t_hbm = 2 * B * n * n * es / (HBM * 1e9)
                t_cmp = B * R * fpu(n) / (PEAK[dt] * 1e12)
                row["bound"] = "hbm" if t_hbm > t_cmp else "alu"
                for kind in ("specialized", "generic"):
                    st = steps if kind == "specialized" else max(1, steps // 2)
                    ms = time_run(n, dt, B, R, x, y, kind, st, 1, stream)
                    ups = B * R / (ms / 1e3)
                    tf = ups * fpu(n) / 1e12
                    gbs = 2 * B * n * n * es / (ms / 1e3) / 1e9
                    row[kind] = {"ms": ms, "updates_per_s": ups, "tflops": tf, "hbm_gbs": gbs,
                                 "frac_hbm": gbs / HBM, "frac_pipe": tf / PEAK[dt]}
                row["speedup"] = row["specialized"]["updates_per_s"] / row["generic"]["updates_per_s"]
                emit(row, fh)
            del x, y
            torch.cuda.empty_cache()


def c4(fh, stream):
    rng = np.random.Generator(np.random.PCG64(1904))
    ns = rng.integers(2, 65, size=1 << 18)
    counts = np.bincount(ns, minlength=65)
    for dt in ("f64", "f32"):
        jm.jit_mat_shutdown()
        jm.jit_mat_init(0)
        jm.jit_mat_set_stream(stream.cuda_stream)
        jm.jit_mat_reset_stats()
        tdt = torch.float64 if dt == "f64" else torch.float32
        groups = []
        for n in range(2, 65):
            if counts[n]:
                x = torch.empty(int(counts[n]), n, n, dtype=tdt, device="cuda")
                jm.jit_mat_fill(n, dt, 1, SEED + n, 0, int(counts[n]), x.data_ptr())
                groups.append((n, int(counts[n]), x, torch.empty_like(x)))
        torch.cuda.synchronize()
        R = 10

        def one_pass(kind, many=True):
            if many:   # one jit_mat_run_many call: parallel compiles + concurrent groups
                jm.jit_mat_run_many([dict(n=n, dtype=dt, batch=b, repeat=R, in_ptr=x.data_ptr(),
                                          out_ptr=y.data_ptr(), kind=kind) for n, b, x, y in groups],
                                    stream=stream.cuda_stream)
                return
            for n, b, x, y in groups:
                jm.jit_mat_run_ex(n, dt, b, R, x.data_ptr(), y.data_ptr(), kind=kind, stream=stream.cuda_stream)

        t0 = time.perf_counter()
        one_pass("specialized", many=False)     # cold, one key after another
        stream.synchronize()
        cold_s = time.perf_counter() - t0
        st = jm.jit_mat_stats()
        keys = [k for k in jm.jit_mat_key_info() if k["kind"] == 0]
        # cold again through jit_mat_run_many (every key compiles in parallel)
        jm.jit_mat_shutdown()
        jm.jit_mat_init(0)
        jm.jit_mat_set_stream(stream.cuda_stream)
        t0 = time.perf_counter()
        one_pass("specialized")
        stream.synchronize()
        par_s = time.perf_counter() - t0
        # cold again, the cold keys compiled as a few multi-expression NVRTC
        # programs (JM_FLAG_BATCH_COMPILE), for several group counts
        batched = {}
        for ng in ("1", "4", str(os.cpu_count() or 8), "16"):
            os.environ["JIT_MAT_COMPILE_GROUPS"] = ng
            jm.jit_mat_shutdown()
            jm.jit_mat_init(0)
            jm.jit_mat_set_stream(stream.cuda_stream)
            jm.jit_mat_reset_stats()
            t0 = time.perf_counter()
            jm.jit_mat_run_many([dict(n=n, dtype=dt, batch=b, repeat=R, in_ptr=x.data_ptr(),
                                      out_ptr=y.data_ptr()) for n, b, x, y in groups],
                                stream=stream.cuda_stream, batch_compile=True)
            stream.synchronize()
            batched[ng] = {"cold_pass_s": time.perf_counter() - t0, "programs": jm.jit_mat_stats()["programs"],
                               "compilations": jm.jit_mat_stats()["compilations"]}
        os.environ.pop("JIT_MAT_COMPILE_GROUPS", None)
        res = {}
        for kind, many in (("specialized", True), ("generic", True), ("specialized_serial", False)):
            kind_ = kind.split("_")[0]
            one_pass(kind_, many)
            stream.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(3):
                one_pass(kind_, many)
            e1.record(stream)
            e1.synchronize()
            ms = e0.elapsed_time(e1) / 3
            tot_updates = int(counts.sum()) * R
            flops = sum(int(counts[n]) * fpu(n) for n in range(65)) * R
            res[kind] = {"ms": ms, "updates_per_s": tot_updates / (ms / 1e3), "tflops": flops / (ms / 1e3) / 1e12}
        emit({"config": "C4", "dtype": dt, "matrices": int(counts.sum()), "keys": len(groups), "repeat": R,
              "cold_pass_s_incl_compiles": cold_s, "compilations": st["compilations"],
              "compile_ms_total_serial": st["compile_ms_total"],
              "compile_ms_per_key_median": float(np.median([k["compile_ms"] for k in keys])),
              "compile_ms_per_key_max": float(np.max([k["compile_ms"] for k in keys])),
              "cold_pass_s_run_many_parallel_compiles": par_s,
              "cold_pass_run_many_batched_programs": batched, "host_cpus": os.cpu_count(),
              "warm": res, "specialized_speedup": res["specialized"]["updates_per_s"] / res["generic"]["updates_per_s"]},
             fh)
        del groups
        torch.cuda.empty_cache()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="c1,c3,c4")
    ap.add_argument("--out", default=None)
    ap.add_argument("--sizes", default="2,3,4,8,16,32,64")
    ap.add_argument("--dtypes", default="f64,f32")
    ap.add_argument("--repeats", default="1,100")
    ap.add_argument("--steps", type=int, default=3)
    a = ap.parse_args()
    torch.cuda.init()
    jm.jit_mat_init(0)
    stream = torch.cuda.Stream()
    jm.jit_mat_set_stream(stream.cuda_stream)
    fh = open(a.out, "a") if a.out else None
    only = a.only.split(",")
    if "c1" in only:
        c1(fh, stream)
    if "c3" in only:
        c3(fh, stream, [int(s) for s in a.sizes.split(",")], a.dtypes.split(","),
           [int(r) for r in a.repeats.split(",")], a.steps)
    if "c4" in only:
        c4(fh, stream)


if __name__ == "__main__":
    main()
