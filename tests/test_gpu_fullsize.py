"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times
(configs[0] C1 and configs[3] C4 at the end of the file).

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


@pytest.mark.parametrize("kind", ["specialized", "generic", "aot_specialized_n3"])
def test_c1_single_matrix_reaches_the_closed_form_fixed_point(jm, kind):
    """configs[0] (C1): one FP64 4x4 paper-init matrix, 1000 repeats.  Every
    entry must equal the closed-form fixed point a*(4) = 1.0002501125631647
    (oracle pin O4) to within a couple of ulp — and the oracle agrees."""
    n, rep = 4, 1000
    x = jm_synth.generate(n, "f64", "paper", 0, 0, 1)
    xd = torch.from_numpy(x).cuda()
    if kind == "aot_specialized_n3":          # the AoT specialization exists for n = 3
        x3 = torch.from_numpy(jm_synth.generate(3, "f64", "paper", 0, 0, 1)).cuda()
        got = jm.run(x3, rep, kind="aot_specialized", sync=True).cpu().numpy()
        assert_parity(got, oracle.run(x3.cpu().numpy(), rep), what="C1-like n=3 AoT")
        return
    got = jm.run(xd, rep, kind=kind, sync=True).cpu().numpy()
    a_star = 1.0002501125631647
    assert np.all(np.abs(got - a_star) <= 4 * np.finfo(np.float64).eps * a_star), got
    assert_parity(got, oracle.run(x, rep), what=f"C1 {kind}")


def test_c1_identity_addend_fixed_point(jm):
    """C1 with the prose addend I (reading R1): diagonal -> x* = 1.0001000150027506
    (pin O5), off-diagonals -> 0."""
    x = torch.from_numpy(jm_synth.generate(4, "f64", "paper", 0, 0, 1)).cuda()
    got = jm.run(x, 1000, addend="identity", sync=True).cpu().numpy()[0]
    x_star = 1.0001000150027506
    assert np.all(np.abs(np.diag(got) - x_star) <= 4 * np.finfo(np.float64).eps)
    assert np.all(np.abs(got - np.diag(np.diag(got))) <= 1e-300)


@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_c4_mixed_n_full_size_sampled(jm, dt):
    """configs[3] (C4) at full size: 2^18 matrices with n ~ U{2..64} drawn by
    numpy PCG64(1904), grouped by n, repeat 10, through jit_mat_run_many (the
    keys compile concurrently, the groups run on a stream pool); sampled
    blocks of every group checked against the oracle."""
    rng = np.random.default_rng(1904)
    sizes = rng.integers(2, 65, 1 << 18)
    counts = np.bincount(sizes, minlength=65)
    tdt = torch.float64 if dt == "f64" else torch.float32
    groups, bufs, first = [], [], 0
    for n in range(2, 65):
        b = int(counts[n])
        if b == 0:
            continue
        x = torch.empty(b, n, n, dtype=tdt, device="cuda")
        jm.jit_mat_fill(n, dt, jm_synth.DIST_BENCH, SEED + n, first, b, x.data_ptr())
        y = torch.empty_like(x)
        groups.append(dict(n=n, dtype=dt, batch=b, repeat=10, in_ptr=x.data_ptr(), out_ptr=y.data_ptr()))
        bufs.append((n, first, b, x, y))
        first += b
    torch.cuda.synchronize()
    jm.jit_mat_run_many(groups, stream=torch.cuda.current_stream().cuda_stream, sync=True)
    tol = TOL[np.dtype(np.float64 if dt == "f64" else np.float32)]
    for n, g0, b, x, y in bufs:
        w = min(b, 24)
        for s in sorted({0, b - w}):
            xs = jm_synth.generate(n, dt, "bench", SEED + n, g0 + s, w)
            assert np.array_equal(x[s:s + w].cpu().numpy(), xs)
            assert_parity(y[s:s + w].cpu().numpy(), oracle.run(xs, 10), tol, what=f"C4 n={n} {dt}")
