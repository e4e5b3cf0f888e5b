"""bench.py's N > 1 path on one GPU: two ranks (gloo record gather, both on the
same device) run jit_mat_run on their own slices; the strong-scaling global
checksum must equal the one-rank run bit for bit."""
from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BENCH = os.path.join(ROOT, "bench.py")

pytestmark = pytest.mark.gpu


def _run(gpus, extra_env=None):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env.update(extra_env or {})
    cmd = [sys.executable, BENCH, "--gpus", str(gpus), "--steps", "2", "--warmup", "3", "--n", "8",
           "--global-batch", "200003", "--repeat", "3", "--no-e2e", "--no-cpu", "--no-generic"]
    p = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stderr[-3000:]
    return json.loads([ln for ln in p.stdout.splitlines() if ln.startswith("{")][-1])


@pytest.mark.timeout(1200)
def test_bench_two_ranks_match_one():
    one = _run(1)
    two = _run(2, {"JM_BENCH_DIST_BACKEND": "gloo"})
    assert one["n_gpus"] == 1 and two["n_gpus"] == 2
    assert two["collective_backend"] == "gloo" and "gloo broadcast" in two["specializations"]
    assert one["checksum_u64"] == two["checksum_u64"]
    assert two["config"]["global_batch"] == 200003 and two["scaling"] == "strong"
    assert two["gpu_launches"] >= 2
