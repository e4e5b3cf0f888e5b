"""Out-of-bounds WRITE checks with guard bands (r02).

compute-sanitizer is closed on this pool in r02, so every kernel kind that
writes through a ragged tail is also run on buffers that are views into a
larger allocation whose guard regions hold a sentinel bit pattern; after the
call the guards must be bit-for-bit intact and the result must still match the
oracle-checked reference run on an unguarded buffer (bitwise: same kernel,
same inputs).  Covers the r02 kinds: the Laghos mass action's tensor-core
kernel (ragged element counts, every Q padding at D = 8, odd D) and the FP32
shifted 16-B staging of odd n >= 55, plus one kernel of every other family.
"""
from __future__ import annotations

import numpy as np
import pytest

import jm_synth

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

SENT64, SENT32 = 0x7FF4DEADBEEF0001, 0x7FA0BEEF   # signalling-NaN payloads no kernel produces


@pytest.fixture(scope="module")
def jm():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1904_08555_b200 as jm
    torch.cuda.init()
    jm.jit_mat_init(0)
    return jm


def _guarded(shape, dtype, guard):
    """(whole, view): view = whole[guard:guard+shape[0]], the rest a sentinel."""
    whole = torch.empty((shape[0] + 2 * guard,) + tuple(shape[1:]), dtype=dtype, device="cuda")
    whole.view(torch.int64 if dtype == torch.float64 else torch.int32).fill_(
        SENT64 if dtype == torch.float64 else SENT32)
    return whole, whole[guard:guard + shape[0]]


def _guards_intact(whole, guard):
    bits = whole.view(torch.int64 if whole.dtype == torch.float64 else torch.int32)
    want = SENT64 if whole.dtype == torch.float64 else SENT32
    head, tail = bits[:guard], bits[guard + (bits.shape[0] - 2 * guard):]
    return bool((head == want).all()) and bool((tail == want).all())


@pytest.mark.parametrize("D,Q,E", [(8, 8, 37), (8, 3, 5), (8, 1, 9), (7, 6, 13), (6, 8, 1), (5, 5, 11),
                                   (4, 4, 67), (2, 8, 3)])
def test_mass_writes_stay_in_bounds(jm, D, Q, E):
    G = 4
    rng = np.random.default_rng(D * 100 + Q * 10 + E)
    B = torch.from_numpy(rng.uniform(-1, 1, (Q, D))).cuda()
    op = torch.from_numpy(rng.uniform(0.5, 2.0, (E, Q, Q))).cuda()
    x = torch.from_numpy(rng.uniform(-1, 1, (E, D, D))).cuda()
    y0 = torch.from_numpy(rng.uniform(-1, 1, (E, D, D))).cuda()
    ref = y0.clone()
    jm.mass(B, op, x, ref, sync=True)
    whole, y = _guarded((E, D, D), torch.float64, G)
    y.copy_(y0)
    jm.mass(B, op, x, y, sync=True)
    assert _guards_intact(whole, G)
    assert torch.equal(y, ref)


@pytest.mark.parametrize("n,dt,R,variant", [(55, "f32", 1, "streaming"), (63, "f32", 1, "streaming"),
                                            (57, "f32", 2, "streaming"), (17, "f32", 1, "streaming"),
                                            (16, "f32", 1, "streaming"), (17, "f64", 3, "resident"),
                                            (33, "f64", 1, "streaming"), (5, "f64", 2, "resident"),
                                            # the tensor-core FP32 kind: padded last m-tile (40), zero-padded
                                            # ragged rows (37, 47, 63), two warps per matrix (57, 64)
                                            (37, "f32", 3, "resident"), (40, "f32", 3, "resident"),
                                            (47, "f32", 3, "resident"), (57, "f32", 3, "resident"),
                                            (63, "f32", 3, "resident"), (64, "f32", 3, "resident")])
def test_update_writes_stay_in_bounds(jm, n, dt, R, variant):
    G, batch = 4, 37   # 4 guard matrices keep the view 16-B aligned for odd n
    tdt = torch.float64 if dt == "f64" else torch.float32
    x = torch.from_numpy(jm_synth.generate(n, dt, "hard", jm_synth.SEED_HARD_BASE + n, 0, batch)).cuda()
    ref = jm.run(x, R, variant=variant, sync=True)
    whole, out = _guarded((batch, n, n), tdt, G)
    jm.run(x, R, out, variant=variant, sync=True)
    assert _guards_intact(whole, G)
    assert torch.equal(out, ref)
