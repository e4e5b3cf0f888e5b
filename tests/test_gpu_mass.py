"""GPU parity of the Laghos 2D mass action (Listing 12 / Fig. 7) vs the oracle."""
from __future__ import annotations

import numpy as np
import pytest

import oracle

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


def _case(D, Q, E, seed):
    rng = np.random.default_rng(seed)
    return (rng.uniform(-1, 1, (Q, D)), rng.uniform(0.5, 2.0, (E, Q, Q)),
            rng.uniform(-1, 1, (E, D, D)), rng.uniform(-1, 1, (E, D, D)))


def _check(got, want, B, op, x, y):
    # error relative to the magnitude scale of the contraction (cf. reading R17)
    absB = np.abs(B)
    s = np.einsum("ad,be,nde->nab", absB, absB, np.abs(x)) * np.abs(op)
    scale = np.max(np.abs(y) + np.einsum("ad,be,nab->nde", absB, absB, s), axis=(1, 2))
    err = np.max(np.abs(got - want), axis=(1, 2)) / scale
    assert float(np.max(err)) <= 1e-12, float(np.max(err))


@pytest.mark.parametrize("kind", ["specialized", "generic"])
@pytest.mark.parametrize("D,Q", [(1, 1), (2, 2), (2, 4), (2, 8), (4, 2), (4, 4), (4, 8), (8, 2),
                                 (8, 4), (8, 8), (3, 5), (5, 3), (7, 6),
                                 # r02 DMMA kernel (jm_plan.h mass_dmma): every Q padding at D = 8
                                 (8, 1), (8, 3), (8, 5), (8, 6), (8, 7), (6, 8), (6, 6)])
def test_mass_parity(jm, D, Q, kind):
    E = 1000 + 37
    B, op, x, y = _case(D, Q, E, 10 * D + Q)
    want = oracle.mass_apply(y, B, op, x)
    tB, to, tx, ty = (torch.from_numpy(a).cuda() for a in (B, op, x, y))
    jm.mass(tB, to, tx, ty, kind=kind, sync=True)
    _check(ty.cpu().numpy(), want, B, op, x, y)


def test_mass_errors_and_cache(jm):
    B, op, x, y = (torch.from_numpy(a).cuda() for a in _case(2, 4, 10, 1))
    lib = jm.lib
    assert lib.jit_mat_mass(9, 4, 0, 10, B.data_ptr(), op.data_ptr(), x.data_ptr(), y.data_ptr(), None) == jm.JM_E_UNSUPPORTED
    assert lib.jit_mat_mass(0, 4, 0, 10, B.data_ptr(), op.data_ptr(), x.data_ptr(), y.data_ptr(), None) == jm.JM_E_INVALID
    assert lib.jit_mat_mass(2, 4, 2, 10, B.data_ptr(), op.data_ptr(), x.data_ptr(), y.data_ptr(), None) == jm.JM_E_UNSUPPORTED
    assert lib.jit_mat_mass(2, 4, 0, 10, B.data_ptr(), op.data_ptr(), x.data_ptr(), x.data_ptr(), None) == jm.JM_E_INVALID
    assert lib.jit_mat_mass(2, 4, 0, 0, None, None, None, None, None) == jm.JM_OK
    st0 = jm.jit_mat_stats()
    for _ in range(20):
        jm.mass(B, op, x, y)
    torch.cuda.synchronize()
    st1 = jm.jit_mat_stats()
    assert st1["compilations"] - st0["compilations"] <= 1


@pytest.mark.parametrize("E", [1, 3, 7, 8, 9, 4096 + 5])
@pytest.mark.parametrize("D,Q", [(8, 8), (8, 3)])
def test_mass_parity_ragged(jm, D, Q, E):
    """element counts below / around one CTA chunk (the DMMA kernel: 8 elements
    per CTA, the next element's loads prefetched) and a ragged large tail"""
    B, op, x, y = _case(D, Q, E, 1000 + E)
    want = oracle.mass_apply(y, B, op, x)
    tB, to, tx, ty = (torch.from_numpy(a).cuda() for a in (B, op, x, y))
    jm.mass(tB, to, tx, ty, sync=True)
    _check(ty.cpu().numpy(), want, B, op, x, y)
