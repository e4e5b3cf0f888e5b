"""GPU parity of the batched multiply-accumulate (Listing 8) vs the oracle."""
from __future__ import annotations

import numpy as np
import pytest

import jm_synth
import oracle

from ._parity import TOL, assert_parity


def assert_mm_parity(got, want, a, b, c, what=""):
    """Error relative to the dot-product scale max(|C| + |A||B|) per matrix (the
    forward-error bound of c + a@b); a plain |result| normalisation is
    meaningless under cancellation (n = 1: c ~ -a*b)."""
    scale = np.max(np.abs(c) + np.abs(a).astype(np.float64) @ np.abs(b).astype(np.float64), axis=(1, 2))
    err = np.max(np.abs(got.astype(np.float64) - want), axis=(1, 2)) / np.where(scale == 0, 1, scale)
    tol = TOL[np.asarray(want).dtype]
    assert float(np.max(err)) <= tol, f"{what}: {float(np.max(err)):.3e} > {tol}"

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def jm():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1904_08555_b200 as jm
    torch.cuda.init()
    jm.jit_mat_init(0)
    return jm


def _inputs(n, dt, batch, seed):
    a = jm_synth.generate(n, dt, "bench", seed, 0, batch)
    b = jm_synth.generate(n, dt, "bench", seed + 1, 0, batch)
    c = jm_synth.generate(n, dt, "bench", seed + 2, 0, batch)
    return a, b, c


@pytest.mark.parametrize("dt", ["f64", "f32"])
@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 7, 8, 9, 15, 16, 17, 31, 32, 33, 64])
@pytest.mark.parametrize("kind", ["specialized", "generic"])
def test_matmul_parity(jm, n, dt, kind):
    batch = {1: 1000, 2: 777, 3: 301}.get(n, 130 if n <= 16 else 9)
    a, b, c = _inputs(n, dt, batch, 100 + n)
    want = oracle.matmul_acc(c, a, b)
    ta, tb, tc = (torch.from_numpy(x).cuda() for x in (a, b, c))
    jm.matmul(ta, tb, tc, kind=kind, sync=True)
    assert_mm_parity(tc.cpu().numpy(), want, a, b, c, what=f"matmul n={n} {dt} {kind}")


@pytest.mark.parametrize("batch", [1, 63, 64, 65, 100_003])
def test_matmul_ragged_and_repeated(jm, batch):
    n = 2
    a, b, c = _inputs(n, "f64", batch, 7)
    ta, tb, tc = (torch.from_numpy(x).cuda() for x in (a, b, c))
    for _ in range(3):                      # the benchmark accumulates over repeats
        jm.matmul(ta, tb, tc)
    torch.cuda.synchronize()
    want = c
    for _ in range(3):
        want = oracle.matmul_acc(want, a, b)
    assert_parity(tc.cpu().numpy(), want, what=f"ragged batch={batch}")   # f64, no cancellation at 1e-12


def test_matmul_aliased_inputs_and_errors(jm):
    n = 8
    a, _, c = _inputs(n, "f64", 50, 3)
    ta, tc = torch.from_numpy(a).cuda(), torch.from_numpy(c).cuda()
    jm.matmul(ta, ta, tc, sync=True)        # a == b allowed: c += a @ a
    assert_mm_parity(tc.cpu().numpy(), oracle.matmul_acc(c, a, a), a, a, c, what="a==b")
    p = ta.data_ptr()
    assert jm.lib.jit_mat_matmul(n, 1, 0, 50, p, p, p, None) == jm.JM_E_INVALID      # c overlaps a
    assert jm.lib.jit_mat_matmul(n, 1, 0, 50, p + 8, p, tc.data_ptr(), None) == jm.JM_E_ALIGN
    assert jm.lib.jit_mat_matmul(n, 1, 2, 50, p, p, tc.data_ptr(), None) == jm.JM_E_UNSUPPORTED
    assert jm.lib.jit_mat_matmul(0, 1, 0, 50, p, p, tc.data_ptr(), None) == jm.JM_E_INVALID
    assert jm.lib.jit_mat_matmul(n, 1, 0, 0, None, None, None, None) == jm.JM_OK


def test_matmul_specialization_is_cached(jm):
    n = 5
    a, b, c = _inputs(n, "f32", 40, 9)
    ta, tb, tc = (torch.from_numpy(x).cuda() for x in (a, b, c))
    st0 = jm.jit_mat_stats()
    for _ in range(50):
        jm.matmul(ta, tb, tc)
    torch.cuda.synchronize()
    st1 = jm.jit_mat_stats()
    assert st1["compilations"] - st0["compilations"] <= 1
    assert st1["hits"] - st0["hits"] >= 49
    info = [k for k in jm.jit_mat_key_info() if k["op"] == 1 and k["n"] == n]
    assert info and info[0]["tile_name"] == "matmul"


def test_lookup_hit_cost_is_small(jm):
    jm.jit_mat_prepare(16, "double")
    ns = jm.jit_mat_time_lookup(16, "double", iters=200_000)
    assert 0 < ns < 1000, ns


@pytest.mark.parametrize("n,dt,batch", [(2, "f64", (1 << 20) + 13), (8, "f32", 300_001), (16, "f64", 60_007),
                                        (33, "f32", 2_003), (1, "f32", 5_000_001), (64, "f64", 701),
                                        (63, "f64", 301), (63, "f32", 150)])
def test_matmul_bulk_ring_wraps(jm, n, dt, batch):
    """Batches large enough that every CTA cycles its bulk-copy ring many times
    (chunks per CTA >> MM_STAGES) plus a ragged tail; checked on a sample of
    matrices (each matrix is independent, R16) including the first, the last and
    the whole tail.  n = 63 has no ring (chunk too large): the staged loop."""
    a, b, c = _inputs(n, dt, batch, 55 + n)
    ta, tb, tc = (torch.from_numpy(x).cuda() for x in (a, b, c))
    jm.matmul(ta, tb, tc, sync=True)
    rng = np.random.default_rng(n)
    idx = np.unique(np.concatenate([rng.integers(0, batch, 2000), np.arange(max(0, batch - 300), batch), [0]]))
    got = tc[torch.from_numpy(idx).cuda()].cpu().numpy()
    want = oracle.matmul_acc(c[idx], a[idx], b[idx])
    assert_mm_parity(got, want, a[idx], b[idx], c[idx], what=f"bulk ring n={n} {dt} batch={batch}")
