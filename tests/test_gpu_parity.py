"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle.

Every case runs on seeded synthetic inputs (jm_synth), is computed by the
oracle on the host, and is compared element by element with the normwise
protocol of SURVEY.md §8(c) (tests/_parity.py).  Inputs are "parity-hard"
(entries U[0,1)*2*4000/n, c*rho = 0.2) at R in {1,2,3,7} — small R where a
wrong product is not washed out by convergence to the fixed point (O4) — plus
paper-init, divergence (O12) and the full-size C2 launch on sampled outputs.
"""
from __future__ import annotations

import numpy as np
import pytest

import jm_synth
import oracle

from ._parity import TOL, assert_parity, max_rel_err

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def jm():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1904_08555_b200 as jm
    torch.cuda.init()
    jm.jit_mat_init(0)
    jm.jit_mat_set_stream(torch.cuda.current_stream().cuda_stream)
    return jm


def _batch_for(n):
    # several CTA chunks plus a ragged tail for every tiling kind
    if n <= 8:
        return 2 * 128 + 37
    if n <= 32:
        return 4 * 9 + 3
    return 7


def _gpu_run(jm, x, repeat, addend="ones", kind="specialized", inplace=False):
    xd = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    out = xd if inplace else torch.empty_like(xd)
    jm.run(xd, repeat, out, addend=addend, kind=kind, sync=True)
    return out.cpu().numpy()


ALL_N = list(range(1, 65))


@pytest.mark.parametrize("dt", ["f64", "f32"])
@pytest.mark.parametrize("n", ALL_N)
def test_parity_hard_ones_all_n(jm, n, dt):
    x = jm_synth.generate(n, dt, "hard", jm_synth.SEED_HARD_BASE + n, 0, _batch_for(n))
    for r in (1, 2, 3, 7):
        want = oracle.run(x, r)
        for kind in ("specialized", "generic"):
            got = _gpu_run(jm, x, r, kind=kind)
            assert_parity(got, want, what=f"n={n} {dt} R={r} {kind}")


@pytest.mark.parametrize("dt", ["f64", "f32"])
@pytest.mark.parametrize("n", ALL_N)
def test_parity_signed_hard_all_n(jm, n, dt):
    """Signed parity-hard inputs (entries U[-1,1)*2*4000/n):
    the products cancel, so a sign error or a dropped term in a path only some
    n take (thin border, staged product, row panels, tiles) is not hidden by
    the all-positive "hard" inputs.  Both kernel variants are forced."""
    x = jm_synth.generate(n, dt, "shard", jm_synth.SEED_HARD_BASE + 1000 + n, 0, _batch_for(n))
    for r in (1, 2, 3):
        want = oracle.run(x, r)
        for kind, variant in (("specialized", "resident"), ("specialized", "streaming"), ("generic", None)):
            xd = torch.from_numpy(np.ascontiguousarray(x)).cuda()
            got = jm.run(xd, r, addend="ones", kind=kind, sync=True, variant=variant).cpu().numpy()
            assert_parity(got, want, what=f"signed n={n} {dt} R={r} {kind} {variant}")
        want_i = oracle.run(x, r, "identity")
        got_i = _gpu_run(jm, x, r, addend="identity")
        assert_parity(got_i, want_i, what=f"signed identity n={n} {dt} R={r}")


IDLE_LANE_SHAPES = [("f64", 17), ("f64", 18), ("f32", 17), ("f32", 18), ("f32", 25), ("f32", 41), ("f32", 42),
                    ("f32", 49), ("f32", 50), ("f32", 51), ("f32", 52), ("f32", 54), ("f32", 55)]


@pytest.mark.parametrize("dt,n", IDLE_LANE_SHAPES)
def test_parity_register_tiles_many_chunks(jm, dt, n):
    """The register-tile shapes whose matrices do not fill a warp (6-, 10-,
    28- and 56-thread matrices: idle lanes, or with JM_TILE_PACK_ALL the
    lane-packed CTA of jm_plan.h F32T.pack, profiles/r02_ab_lane_pack.md):
    several whole CTA chunks (up to 85 matrices each) plus a ragged tail, both
    signs, resident kernel, in place as well."""
    batch = 3 * 85 + 5 if n <= 25 else 3 * 8 + 5
    for dist, seed in (("hard", 2000), ("shard", 3000)):
        x = jm_synth.generate(n, dt, dist, jm_synth.SEED_HARD_BASE + seed + n, 0, batch)
        for r in (1, 2, 5):
            want = oracle.run(x, r)
            xd = torch.from_numpy(np.ascontiguousarray(x)).cuda()
            got = jm.run(xd, r, addend="ones", sync=True, variant="resident").cpu().numpy()
            assert_parity(got, want, what=f"packed {dist} n={n} {dt} R={r}")
        jm.run(xd, 3, xd, addend="identity", sync=True, variant="resident")
        assert_parity(xd.cpu().numpy(), oracle.run(x, 3, "identity"), what=f"packed in-place n={n} {dt}")


@pytest.mark.parametrize("dt", ["f64", "f32"])
@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 7, 8, 9, 13, 16, 17, 24, 32, 33, 40, 48, 57, 64])
def test_parity_identity_addend(jm, n, dt):
    x = jm_synth.generate(n, dt, "hard", jm_synth.SEED_HARD_BASE + n, 0, _batch_for(n))
    for r in (1, 3, 40):
        want = oracle.run(x, r, "identity")
        for kind in ("specialized", "generic"):
            got = _gpu_run(jm, x, r, addend="identity", kind=kind)
            assert_parity(got, want, what=f"identity n={n} {dt} R={r} {kind}")


@pytest.mark.parametrize("dt", ["f64", "f32"])
@pytest.mark.parametrize("n", [1, 2, 3, 4, 6, 8, 12, 16, 20, 32, 34])
def test_parity_paper_init(jm, n, dt):
    # PAPER.md Listing 4/5: m(i,j) = i + size*j, the benchmark's own input
    x = jm_synth.generate(n, dt, "paper", 0, 0, 3)
    for r in (1, 2, 20):
        want = oracle.run(x, r)
        got = _gpu_run(jm, x, r)
        assert_parity(got, want, what=f"paper n={n} {dt} R={r}")


@pytest.mark.parametrize("n,rep", [(35, 14), (48, 10), (64, 9)])
@pytest.mark.parametrize("kind", ["specialized", "generic"])
def test_divergence_to_inf(jm, n, rep, kind):
    # O12: paper-init n >= 35 reaches +inf everywhere, no NaN
    x = jm_synth.generate(n, "f64", "paper", 0, 0, 2)
    got = _gpu_run(jm, x, rep, kind=kind)
    assert np.all(np.isposinf(got))
    for r in (1, 2, 3):
        assert_parity(_gpu_run(jm, x, r, kind=kind), oracle.run(x, r), what=f"pre-divergence R={r}")


@pytest.mark.parametrize("n", [17, 24, 32, 33, 37, 40, 47, 48, 57, 63, 64])
def test_f32_overflow_positions_match(jm, n):
    # FP32 paper init overflows within a few updates at these n; the tiles pad
    # to multiples of 8 / 4, and the padding must never leak NaN or inf into
    # the real entries: every non-finite position must match the oracle's.
    x = jm_synth.generate(n, "f32", "paper", 0, 0, 3)
    for r in (1, 2, 4, 8, 16):
        assert_parity(_gpu_run(jm, x, r), oracle.run(x, r), what=f"f32 paper n={n} R={r}")


@pytest.mark.parametrize("dt", ["f64", "f32"])
@pytest.mark.parametrize("n", [1, 3, 4, 5, 8, 16, 33, 64])
def test_repeat_zero_is_bitwise_copy(jm, n, dt):
    x = jm_synth.generate(n, dt, "bench", jm_synth.SEED_BENCH, 0, _batch_for(n))
    for kind in ("specialized", "generic"):
        assert np.array_equal(_gpu_run(jm, x, 0, kind=kind), x)


@pytest.mark.parametrize("dt", ["f64", "f32"])
@pytest.mark.parametrize("n", [2, 3, 5, 8, 16, 31, 40])
def test_in_place_alias(jm, n, dt):
    x = jm_synth.generate(n, dt, "hard", 7, 0, _batch_for(n))
    want = oracle.run(x, 2)
    assert_parity(_gpu_run(jm, x, 2, inplace=True), want, what=f"in-place n={n} {dt}")


@pytest.mark.parametrize("n,dt", [(2, "f64"), (3, "f64"), (4, "f32"), (7, "f32"), (8, "f64"), (16, "f64"),
                                  (13, "f64"), (20, "f32"), (64, "f64"), (45, "f32")])
@pytest.mark.parametrize("batch", [1, 31, 32, 33, 1000, (1 << 16) + 7])
def test_ragged_batches(jm, n, dt, batch):
    if batch > 5000 and n > 16:
        batch = 4099
    x = jm_synth.generate(n, dt, "hard", 11, 0, batch)
    idx = np.unique(np.r_[0:min(batch, 64), max(0, batch - 64):batch,
                          np.random.default_rng(1).integers(0, batch, 128)])
    want = oracle.run(x[idx], 3)
    got = _gpu_run(jm, x, 3)[idx]
    assert_parity(got, want, what=f"ragged n={n} {dt} batch={batch}")


def test_batch_zero_is_noop(jm):
    x = torch.zeros(0, 4, 4, dtype=torch.float64, device="cuda")
    jm.run(x, 5, sync=True)


@pytest.mark.parametrize("dt,tol", [("f64", 1e-12), ("f32", 1e-5)])
def test_c2_full_size_sampled(jm, dt, tol):
    """BASELINE.json configs[1] at full size, as bench.py launches it."""
    n, batch, rep = 16, 1 << 20, 100
    tdt = torch.float64 if dt == "f64" else torch.float32
    x = torch.empty(batch, n, n, dtype=tdt, device="cuda")
    jm.jit_mat_fill(n, dt, jm_synth.DIST_BENCH, jm_synth.SEED_BENCH, 0, batch, x.data_ptr())
    out = torch.empty_like(x)
    jm.run(x, rep, out, sync=True)
    rng = np.random.default_rng(2)
    idx = np.unique(np.r_[0:1024, batch - 1024:batch, rng.integers(0, batch, 2048)])
    # regenerate the sampled inputs on the host from the same definition
    xs = np.stack([jm_synth.generate(n, dt, "bench", jm_synth.SEED_BENCH, int(b), 1)[0] for b in idx])
    assert np.array_equal(x[torch.from_numpy(idx).cuda()].cpu().numpy(), xs)
    want = oracle.run(xs, rep)
    got = out[torch.from_numpy(idx).cuda()].cpu().numpy()
    assert_parity(got, want, tol, what=f"C2 {dt}")


@pytest.mark.parametrize("dt", ["f64", "f32"])
@pytest.mark.parametrize("dist", ["paper", "bench", "hard", "shard"])
@pytest.mark.parametrize("n", [1, 3, 16, 64])
def test_device_fill_matches_host_generator(jm, n, dt, dist):
    batch, first = 301, 12345
    tdt = torch.float64 if dt == "f64" else torch.float32
    x = torch.empty(batch, n, n, dtype=tdt, device="cuda")
    jm.jit_mat_fill(n, dt, jm_synth.DISTS[dist], 99, first, batch, x.data_ptr())
    torch.cuda.synchronize()
    assert np.array_equal(x.cpu().numpy(), jm_synth.generate(n, dt, dist, 99, first, batch))


@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_device_checksum_matches_host(jm, dt):
    n, batch, first = 8, 5000, 777
    x = jm_synth.generate(n, dt, "bench", 5, first, batch)
    xd = torch.from_numpy(x).cuda()
    u, f = jm.jit_mat_checksum(n, dt, first, batch, xd.data_ptr())
    assert u == jm_synth.checksum(x, n, first)
    assert f == pytest.approx(float(np.sum(x.astype(np.float64))), rel=1e-9, abs=1e-6)


@pytest.mark.parametrize("n,dt", [(4, "f64"), (16, "f64"), (9, "f32"), (33, "f64")])
def test_host_buffer_path(jm, n, dt, monkeypatch):
    monkeypatch.setenv("JIT_MAT_HOST_CHUNK_MB", "1")   # many chunks: exercise the rotation
    batch = 20000 if n <= 16 else 1500
    x = jm_synth.generate(n, dt, "hard", 3, 0, batch)
    out = np.empty_like(x)
    jm.jit_mat_run_host(n, dt, batch, 3, x.ctypes.data, out.ctypes.data)
    idx = np.r_[0:50, batch - 50:batch]
    assert_parity(out[idx], oracle.run(x[idx], 3), what=f"host path n={n} {dt}")
    # and identical to the device path bit for bit (same kernel)
    assert np.array_equal(out, _gpu_run(jm, x, 3))


def test_specialized_and_generic_agree_closely(jm):
    x = jm_synth.generate(16, "f64", "bench", 1, 0, 64)
    a = _gpu_run(jm, x, 50, kind="specialized")
    b = _gpu_run(jm, x, 50, kind="generic")
    assert max_rel_err(a, b) <= TOL[np.dtype(np.float64)]


def test_run_many_mixed_sizes_matches_single_runs(jm):
    """Mixed-N batch (configs[3]) through jit_mat_run_many == per-group runs, bitwise."""
    rng = np.random.default_rng(5)
    groups, bufs = [], []
    for n in [2, 3, 5, 8, 13, 16, 24, 31, 33, 64]:
        for dt in ("f64", "f32"):
            b = int(rng.integers(1, 300))
            x = torch.from_numpy(jm_synth.generate(n, dt, "hard", 3 + n, 0, b)).cuda()
            y = torch.empty_like(x)
            groups.append(dict(n=n, dtype=dt, batch=b, repeat=3, in_ptr=x.data_ptr(),
                               out_ptr=y.data_ptr(), kind="specialized" if n % 2 else "generic"))
            bufs.append((x, y))
    groups.append(dict(n=7, dtype="f64", batch=0, repeat=3, in_ptr=0, out_ptr=0))
    jm.jit_mat_run_many(groups, stream=torch.cuda.current_stream().cuda_stream, sync=True)
    for (x, y), g in zip(bufs, groups):
        ref = torch.empty_like(x)
        jm.run(x, 3, ref, kind=g["kind"], sync=True)
        assert torch.equal(y, ref), g
        if g["n"] <= 16:
            assert_parity(y.cpu().numpy(), oracle.run(x.cpu().numpy(), 3), what=str(g))


def test_run_many_rejects_bad_descriptor_before_launch(jm):
    x = torch.zeros(4, 4, 4, dtype=torch.float64, device="cuda")
    y = torch.full_like(x, 7.0)
    bad = [dict(n=4, dtype="f64", batch=4, repeat=1, in_ptr=x.data_ptr(), out_ptr=y.data_ptr()),
           dict(n=99, dtype="f64", batch=4, repeat=1, in_ptr=x.data_ptr(), out_ptr=y.data_ptr())]
    with pytest.raises(jm.JitMatError):
        jm.jit_mat_run_many(bad, sync=True)
    torch.cuda.synchronize()
    assert torch.all(y == 7.0)


@pytest.mark.parametrize("dt", ["f64", "f32"])
@pytest.mark.parametrize("n", [1, 2, 3, 4, 5])
def test_latency_variant(jm, n, dt):
    """Tiny batches run a warp per matrix (k_update_lat, C1's kernel): parity
    with the oracle, bit-identical to the thread-per-matrix kernel (same
    summation order), picked automatically for batch <= 4 x SMs."""
    for batch, dist in ((1, "paper"), (7, "shard"), (600, "hard")):
        x = jm_synth.generate(n, dt, dist, 40 + n, 0, batch)
        xd = torch.from_numpy(np.ascontiguousarray(x)).cuda()
        for r in (1, 3, 1000 if batch == 1 else 25):
            got = jm.run(xd, r, sync=True, variant="latency").cpu().numpy()
            tpm = jm.run(xd, r, sync=True, variant="resident").cpu().numpy()
            assert np.array_equal(got.view(np.uint8), tpm.view(np.uint8)), f"lat != tpm n={n} {dt} b={batch} R={r}"
            assert_parity(got, oracle.run(x, r), what=f"latency n={n} {dt} batch={batch} R={r}")
            auto = jm.run(xd, r, sync=True).cpu().numpy()
            assert np.array_equal(auto.view(np.uint8), got.view(np.uint8))
    x = jm_synth.generate(n, dt, "shard", 9, 0, 5)
    xd = torch.from_numpy(x).cuda()
    got_i = jm.run(xd, 3, addend="identity", sync=True, variant="latency").cpu().numpy()
    assert_parity(got_i, oracle.run(x, 3, "identity"), what=f"latency identity n={n} {dt}")
    lat = [k for k in jm.jit_mat_key_info() if k["variant"] == 2 and k["n"] == n]
    assert lat and lat[0]["tile_name"] == "lat"
