"""GPU parity of the STREAMING variant (bulk-copy ring, low repeat) vs the oracle.

The streaming variant runs the same tiling kinds as the resident kernel behind
a TMA bulk-copy ring (jm_update.cuh ``Ring``; jm_plan.h ``plan_stream``), and
the library picks it when repeat * (n + 1) is below the roofline switch point
(include/jit_mat.h VARIANT).  Both variants are forced here for every n that
has one, on parity-hard inputs, with batches that span
several ring chunks and a ragged tail, and at sizes where every CTA walks the
ring through several phase flips.  Where the two variants use the same tile
mapping they do the same arithmetic in the same order and must agree bit for
bit (all sizes but f64 n = 33, 34).
"""
from __future__ import annotations

import numpy as np
import pytest

import jm_synth
import oracle

from ._parity import assert_parity

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

# every size has a low-repeat variant: the bulk-copy ring behind the DMMA /
# FP32 kinds, the double-buffered stage behind thread-per-matrix (n <= 7 / 8)
STREAM_N = {"f64": list(range(1, 65)), "f32": list(range(1, 65))}


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
    # several ring chunks (8 KB-ish each) plus a ragged tail
    return 293 if n <= 12 else (77 if n <= 32 else 9)


# f64 sizes whose resident kernel is the DFMA register tile (jm_plan.h F64T_TABLE)
# and whose low-repeat kernel is the DMMA ring
F64_REG_N = (11, 12, 17, 18, 19, 20)


def _same_bits(n, dt):
    # both variants form every entry in the same order, except f64 n = 33 / 34,
    # where the resident kernel (whole matrix per warp) takes the thin-border
    # DFMA path and the streaming one (one warp per row tile) does not, and
    # f64 n = 9 / 10 and f32 n = 12..14, whose resident kernel is thread per
    # matrix with a staged product (TPMS) and whose low-repeat kernel is the
    # DMMA ring / the row-panel ring, and the DFMA register-tile sizes, and
    # f32 n = 32 and 37..64, whose resident kernel runs on the tensor cores (3xTF32)
    return not ((dt == "f64" and n in (9, 10, 33, 34) + F64_REG_N) or (dt == "f32" and (n in (12, 13, 14, 32) or n >= 37)))


def test_f64_reg_sizes_match_the_plan(jm):
    """F64_REG_N above is the set of sizes the planner gives the DFMA register tiles."""
    got = []
    for n in range(1, 65):
        jm.jit_mat_prepare(n, "double")
    for k in jm.jit_mat_key_info():
        if k["op"] == 0 and k["dtype"] == 1 and k["kind"] == 0 and k["addend"] == 0 and k["variant"] == 0 \
                and k["tile_name"] == "f64_reg":
            got.append(k["n"])
    assert sorted(got) == list(F64_REG_N)


def _run(jm, x, repeat, variant, addend="ones", inplace=False):
    xd = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    out = xd if inplace else torch.empty_like(xd)
    jm.run(xd, repeat, out, addend=addend, sync=True, variant=variant)
    return out.cpu().numpy()


@pytest.mark.parametrize("dt", ["f64", "f32"])
@pytest.mark.parametrize("n", sorted(set(STREAM_N["f64"]) | set(STREAM_N["f32"])))
def test_stream_parity_all_n(jm, n, dt):
    if n not in STREAM_N[dt]:
        pytest.skip("thread-per-matrix size: no streaming variant")
    x = jm_synth.generate(n, dt, "hard", jm_synth.SEED_HARD_BASE + n, 0, _batch_for(n))
    for r in (1, 2, 3):
        want = oracle.run(x, r)
        got_s = _run(jm, x, r, "streaming")
        assert_parity(got_s, want, what=f"streaming n={n} {dt} R={r}")
        got_r = _run(jm, x, r, "resident")
        if _same_bits(n, dt):
            assert np.array_equal(got_s.view(np.uint8), got_r.view(np.uint8)), \
                f"streaming and resident differ bitwise at n={n} {dt} R={r}"
        else:
            assert_parity(got_r, want, what=f"resident n={n} {dt} R={r}")


@pytest.mark.parametrize("dt", ["f64", "f32"])
@pytest.mark.parametrize("n", [9, 16, 17, 24, 33, 40, 57, 64])
def test_stream_identity_addend(jm, n, dt):
    x = jm_synth.generate(n, dt, "hard", jm_synth.SEED_HARD_BASE + n, 0, _batch_for(n))
    for r in (1, 3):
        assert_parity(_run(jm, x, r, "streaming", addend="identity"), oracle.run(x, r, "identity"),
                      what=f"streaming identity n={n} {dt} R={r}")


@pytest.mark.parametrize("n,dt", [(3, "f64"), (4, "f64"), (7, "f64"), (3, "f32"), (8, "f32"),
                                  (8, "f64"), (16, "f64"), (24, "f64"), (32, "f64"), (33, "f64"),
                                  (64, "f64"), (9, "f32"), (16, "f32"), (17, "f32"), (32, "f32"),
                                  (63, "f32"), (64, "f32")])
def test_stream_ring_wraps(jm, n, dt):
    """Batches large enough that every persistent CTA takes many chunks (ring
    phase flips, refills behind bulk stores), checked on sampled outputs."""
    es = 8 if dt == "f64" else 4
    batch = 148 * 48 * max(1, 16384 // (n * n * es)) + 5
    x = jm_synth.generate(n, dt, "hard", 21 + n, 0, batch)
    got = _run(jm, x, 2, "streaming")
    rng = np.random.default_rng(n)
    idx = np.unique(np.r_[0:96, batch - 96:batch, rng.integers(0, batch, 512)])
    assert_parity(got[idx], oracle.run(x[idx], 2), what=f"ring n={n} {dt} batch={batch}")
    res = _run(jm, x, 2, "resident")
    if _same_bits(n, dt):
        assert np.array_equal(got, res)
    else:
        assert_parity(res[idx], oracle.run(x[idx], 2), what=f"ring resident n={n} {dt}")


@pytest.mark.parametrize("n,dt", [(16, "f64"), (40, "f64"), (20, "f32"), (64, "f32")])
def test_stream_in_place(jm, n, dt):
    x = jm_synth.generate(n, dt, "hard", 5, 0, _batch_for(n) * 5)
    assert_parity(_run(jm, x, 1, "streaming", inplace=True), oracle.run(x, 1),
                  what=f"streaming in place n={n} {dt}")


@pytest.mark.parametrize("batch", [1, 2, 3, 5, 17])
def test_stream_tiny_batches(jm, batch):
    # fewer matrices than one chunk: only the ragged (synchronous) path runs
    for n, dt in ((8, "f64"), (33, "f64"), (63, "f32")):
        x = jm_synth.generate(n, dt, "hard", 8, 0, batch)
        assert_parity(_run(jm, x, 1, "streaming"), oracle.run(x, 1), what=f"tiny n={n} {dt} b={batch}")


def test_variant_selection_and_key_info(jm):
    # the default switch: stream iff repeat * (n + 1) < stream_rn(n, dtype)
    assert jm.jit_mat_prepare_for(16, "f64", 1) == 0       # below stream_lo: resident
    assert jm.jit_mat_prepare_for(16, "f64", 2) == 1
    assert jm.jit_mat_prepare_for(16, "f64", 35) == 1      # 595 < 600
    assert jm.jit_mat_prepare_for(16, "f64", 36) == 0      # 612
    assert jm.jit_mat_prepare_for(64, "f64", 6) == 1       # 390 < 400
    assert jm.jit_mat_prepare_for(64, "f64", 7) == 0
    assert jm.jit_mat_prepare_for(33, "f64", 2) == 1       # 68 < 100: thin-border resident above
    assert jm.jit_mat_prepare_for(33, "f64", 3) == 0
    assert jm.jit_mat_prepare_for(15, "f32", 3) == 1       # 48 < 64 (row-panel ring)
    assert jm.jit_mat_prepare_for(15, "f32", 4) == 0
    assert jm.jit_mat_prepare_for(12, "f32", 1) == 0       # TPMS beats the ring even at R = 1
    assert jm.jit_mat_prepare_for(13, "f32", 1) == 1 and jm.jit_mat_prepare_for(13, "f32", 2) == 0
    assert jm.jit_mat_prepare_for(16, "f32", 24) == 1      # n = 16: register tiles, streaming to R = 24
    assert jm.jit_mat_prepare_for(16, "f32", 25) == 0
    # FP32 tiles: stream while R <= F32T_STREAM_MAXR[n] (jm_plan.h f32t_rn)
    assert jm.jit_mat_prepare_for(64, "f32", 3) == 1 and jm.jit_mat_prepare_for(64, "f32", 4) == 0   # (tensor cores above)
    assert jm.jit_mat_prepare_for(47, "f32", 4) == 1 and jm.jit_mat_prepare_for(47, "f32", 5) == 0     # (tensor cores above)
    assert jm.jit_mat_prepare_for(30, "f32", 50) == 1 and jm.jit_mat_prepare_for(30, "f32", 51) == 0
    assert jm.jit_mat_prepare_for(32, "f32", 2) == 1 and jm.jit_mat_prepare_for(32, "f32", 3) == 0   # (tensor cores)
    assert jm.jit_mat_prepare_for(17, "f32", 6) == 1 and jm.jit_mat_prepare_for(17, "f32", 7) == 0
    assert jm.jit_mat_prepare_for(8, "f64", 1) == 0        # n = 8 DMMA: resident (measured)
    assert jm.jit_mat_prepare_for(4, "f64", 1, flags=jm.JM_FLAG_STREAMING) == 1   # TPM: staged variant
    assert jm.jit_mat_prepare_for(4, "f64", 1) == 0        # light TPM sizes stay resident
    assert jm.jit_mat_prepare_for(3, "f32", 7) == 0        # ... except f32 n = 3 from R = 8 on
    assert jm.jit_mat_prepare_for(3, "f32", 8) == 1 and jm.jit_mat_prepare_for(3, "f32", 100) == 1
    assert jm.jit_mat_prepare_for(6, "f64", 1) == 0        # register-heavy TPM: the resident kernel prefetches
    assert jm.jit_mat_prepare_for(16, "f64", 1, kind="generic") == 0
    assert jm.jit_mat_prepare_for(16, "f64", 100, flags=jm.JM_FLAG_STREAMING) == 1
    assert jm.jit_mat_prepare_for(24, "f64", 1) == 1
    assert jm.jit_mat_prepare_for(8, "f64", 100, flags=jm.JM_FLAG_STREAMING) == 1
    assert jm.jit_mat_prepare_for(16, "f64", 1, flags=jm.JM_FLAG_RESIDENT) == 0
    jm.jit_mat_prepare_for(16, "f64", 1)
    info = [k for k in jm.jit_mat_key_info() if k["op"] == 0 and k["n"] == 16 and k["dtype"] == 1
            and k["kind"] == 0 and k["addend"] == 0]
    assert sorted(k["variant"] for k in info) == [0, 1]
    for k in info:
        assert k["state"] == 2 and k["local_bytes"] == 0 and k["tile_name"] == "warp_dmma"


def test_run_many_uses_stream_variant(jm):
    xs, ys, groups = [], [], []
    for n, dt in ((16, "f64"), (32, "f32"), (4, "f64")):
        x = torch.from_numpy(jm_synth.generate(n, dt, "hard", 9, 0, 100)).cuda()
        y = torch.empty_like(x)
        groups.append(dict(n=n, dtype=dt, batch=100, repeat=1, in_ptr=x.data_ptr(), out_ptr=y.data_ptr()))
        xs.append(x)
        ys.append(y)
    jm.jit_mat_run_many(groups, stream=torch.cuda.current_stream().cuda_stream, sync=True)
    for x, y, g in zip(xs, ys, groups):
        assert_parity(y.cpu().numpy(), oracle.run(x.cpu().numpy(), 1), what=str(g))
