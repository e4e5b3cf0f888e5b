"""bench.py launch contract on CPU (no GPU): `--gpus N` without torchrun
re-launches N ranks itself, WORLD_SIZE must equal --gpus, and both arms report
n_gpus = N (VERDICT r01 "make multi-GPU driver-ready")."""
from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BENCH = os.path.join(ROOT, "bench.py")


def _env(**kw):
    e = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    e.update(kw)
    return e


def test_gpus_n_relaunches_n_ranks():
    # (--n: torch.distributed.run's parser would take it for --nnodes; relaunch passes --size)
    p = subprocess.run([sys.executable, BENCH, "--gpus", "2", "--steps", "1", "--warmup", "3", "--n", "8"],
                       env=_env(JM_BENCH_DRY_RUN="1"), capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stderr[-2000:]
    recs = [json.loads(ln) for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert sorted(r["rank"] for r in recs) == [0, 1]
    assert all(r["world"] == 2 and r["gpus"] == 2 for r in recs)


def test_world_size_must_match_gpus():
    p = subprocess.run([sys.executable, BENCH, "--gpus", "4", "--steps", "1"],
                       env=_env(JM_BENCH_DRY_RUN="1", WORLD_SIZE="2", RANK="0", LOCAL_RANK="0"),
                       capture_output=True, text=True, timeout=120)
    assert p.returncode != 0 and "WORLD_SIZE=2" in (p.stderr + p.stdout)


def test_gpus_defaults_to_world_size():
    p = subprocess.run([sys.executable, BENCH, "--steps", "1"],
                       env=_env(JM_BENCH_DRY_RUN="1", WORLD_SIZE="3", RANK="1", LOCAL_RANK="1"),
                       capture_output=True, text=True, timeout=120)
    assert p.returncode == 0, p.stderr[-2000:]
    assert json.loads(p.stdout.strip().splitlines()[-1]) == {"rank": 1, "world": 3, "gpus": 3, "local_rank": 1}


@pytest.mark.timeout(600)
def test_reference_arm_reports_n_gpus():
    """--impl reference --gpus 2 (plain process): rank 0 alone runs the oracle arm, n_gpus = 2."""
    p = subprocess.run([sys.executable, BENCH, "--impl", "reference", "--gpus", "2", "--steps", "1",
                        "--warmup", "3", "--n", "4", "--batch", "256", "--repeat", "2"],
                       env=_env(), capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    line = json.loads(p.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["n_gpus"] == 2 and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "oracle"
