"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times.

configs[2] (C3: N sweep, batch sized to 8 GB of input) and configs[4] (C5:
2^26 FP64 8x8 and 2^22 FP64 32x32 per GPU, repeat 100 and 1) are run at full
size on the device, exactly as bench.py launches them (device fill from the
counter hash, jit_mat_run_ex, the library-chosen variant and grid), and
checked against the CPU oracle on sampled matrices: contiguous blocks at the
start, the end (the ragged tail of the persistent grid) and spread across the
batch, each regenerated on the host from the same counter hash.  For C5 the
order-independent device checksum of the whole output must also be unchanged
when the same global batch runs as two halves (the W = 2 split, SURVEY.md
§8(e)).
"""
from __future__ import annotations

import numpy as np
import pytest

import jm_synth
import oracle

from ._parity import TOL, assert_parity

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

SEED = jm_synth.SEED_BENCH


@pytest.fixture(scope="module")
def jm():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1904_08555_b200 as jm
    torch.cuda.init()
    jm.jit_mat_init(0)
    return jm


def _blocks(batch, rng, nblocks=12, width=48):
    starts = [0, max(0, batch - width)] + list(rng.integers(0, max(1, batch - width), nblocks))
    return sorted({(int(s), int(min(width, batch - s))) for s in starts})


def _run_fullsize(jm, n, dt, batch, repeat):
    tdt = torch.float64 if dt == "f64" else torch.float32
    st = torch.cuda.current_stream()
    jm.jit_mat_set_stream(st.cuda_stream)
    x = torch.empty(batch, n, n, dtype=tdt, device="cuda")
    y = torch.empty_like(x)
    jm.jit_mat_fill(n, dt, jm_synth.DIST_BENCH, SEED, 0, batch, x.data_ptr())
    jm.jit_mat_run_ex(n, dt, batch, repeat, x.data_ptr(), y.data_ptr(), stream=st.cuda_stream)
    st.synchronize()
    return x, y, st


def _check_sampled(jm, x, y, n, dt, batch, repeat, seed):
    rng = np.random.default_rng(seed)
    tol = TOL[np.dtype(np.float64 if dt == "f64" else np.float32)]
    for s, w in _blocks(batch, rng):
        xs = jm_synth.generate(n, dt, "bench", SEED, s, w)
        assert np.array_equal(x[s:s + w].cpu().numpy(), xs)          # device fill == host definition
        assert_parity(y[s:s + w].cpu().numpy(), oracle.run(xs, repeat), tol,
                      what=f"full size n={n} {dt} batch={batch} R={repeat} block {s}+{w}")


@pytest.mark.parametrize("n,dt,repeat", [(2, "f64", 1), (4, "f32", 100), (16, "f32", 1),
                                         (32, "f64", 1), (64, "f64", 100), (64, "f32", 1)])
def test_c3_full_size_sampled(jm, n, dt, repeat):
    """configs[2]: batch = floor(8e9 / (n^2 * sizeof T)) — 8 GB of input."""
    es = 8 if dt == "f64" else 4
    batch = int(8e9 // (n * n * es))
    x, y, _ = _run_fullsize(jm, n, dt, batch, repeat)
    _check_sampled(jm, x, y, n, dt, batch, repeat, seed=n)
    del x, y
    torch.cuda.empty_cache()


@pytest.mark.parametrize("n,batch", [(8, 1 << 26), (32, 1 << 22)])
@pytest.mark.parametrize("repeat", [100, 1])
def test_c5_full_size_sampled_and_split_invariant(jm, n, batch, repeat):
    """configs[4] at W = 1 (34.4 GB in + 34.4 GB out), plus the W = 2 split of
    the same global batch: the order-independent checksum must not change."""
    x, y, st = _run_fullsize(jm, n, "f64", batch, repeat)
    _check_sampled(jm, x, y, n, "f64", batch, repeat, seed=repeat)
    whole, _ = jm.jit_mat_checksum(n, "f64", 0, batch, y.data_ptr())
    half = batch // 2
    y.zero_()
    for first, cnt in ((0, half), (half, batch - half)):         # two "ranks", one device
        jm.jit_mat_run_ex(n, "f64", cnt, repeat, x[first].data_ptr(), y[first].data_ptr(),
                          stream=st.cuda_stream)
    st.synchronize()
    c0, _ = jm.jit_mat_checksum(n, "f64", 0, half, y.data_ptr())
    c1, _ = jm.jit_mat_checksum(n, "f64", half, batch - half, y[half].data_ptr())
    assert (c0 + c1) % (1 << 64) == whole
    del x, y
    torch.cuda.empty_cache()
