"""Pins for the Laghos 2D mass-operator oracle (§5.3, Listing 12; reading R18).

The oracle follows the sum-factorised loop order; these tests check it
against the plain 4-index definition (numpy einsum, a library routine), exact
rational arithmetic on tiny cases, and properties of a mass operator
(identity basis -> pointwise product, symmetry, linearity).
"""
from __future__ import annotations

from fractions import Fraction

import numpy as np
import pytest

import oracle


def _case(D, Q, E, seed):
    rng = np.random.default_rng(seed)
    B = rng.uniform(-1, 1, (Q, D))
    op = rng.uniform(0.5, 2.0, (E, Q, Q))
    x = rng.uniform(-1, 1, (E, D, D))
    y = rng.uniform(-1, 1, (E, D, D))
    return B, op, x, y


def _einsum(B, op, x, y):
    s = np.einsum("ad,be,nde->nab", B, B, x)            # S[qy][qx]
    s = s * op
    return y + np.einsum("ad,be,nab->nde", B, B, s)


@pytest.mark.parametrize("D,Q", [(1, 1), (2, 2), (2, 4), (4, 8), (3, 5), (8, 8), (8, 2)])
def test_matches_four_index_definition(D, Q):
    B, op, x, y = _case(D, Q, 11, D * 10 + Q)
    got = oracle.mass_apply(y, B, op, x)
    want = _einsum(B, op, x, y)
    np.testing.assert_allclose(got, want, rtol=1e-13, atol=1e-13)


def test_exact_rational_tiny():
    D, Q = 2, 3
    B, op, x, y = _case(D, Q, 2, 5)
    got = oracle.mass_apply(y, B, op, x)
    F = np.vectorize(Fraction)
    Bf, opf, xf, yf = F(B), F(op), F(x), F(y)
    for e in range(2):
        S = [[sum(Bf[a][d] * Bf[b][f] * xf[e][d][f] for d in range(D) for f in range(D)) * opf[e][a][b]
              for b in range(Q)] for a in range(Q)]
        for d in range(D):
            for f in range(D):
                exact = yf[e][d][f] + sum(Bf[a][d] * Bf[b][f] * S[a][b] for a in range(Q) for b in range(Q))
                assert abs(got[e, d, f] - float(exact)) <= 64 * np.finfo(float).eps * 8


def test_identity_basis_is_pointwise():
    D = Q = 5
    _, op, x, y = _case(D, Q, 7, 3)
    got = oracle.mass_apply(y, np.eye(D), op, x)
    assert np.array_equal(got, y + op * x)      # every sum has one nonzero term: exact


@pytest.mark.parametrize("D,Q", [(2, 4), (4, 4), (3, 7)])
def test_symmetric_and_linear(D, Q):
    B, op, x1, _ = _case(D, Q, 4, 21)
    x2 = np.random.default_rng(22).uniform(-1, 1, x1.shape)
    z = np.zeros_like(x1)
    a1, a2 = oracle.mass_apply(z, B, op, x1), oracle.mass_apply(z, B, op, x2)
    np.testing.assert_allclose(np.sum(a1 * x2, axis=(1, 2)), np.sum(x1 * a2, axis=(1, 2)), rtol=1e-12)
    np.testing.assert_allclose(oracle.mass_apply(z, B, op, 2 * x1 - x2), 2 * a1 - a2, rtol=1e-12, atol=1e-14)


def test_one_by_one_closed_form():
    B = np.array([[1.5]])
    op = np.array([[[2.0]]])
    x = np.array([[[3.0]]])
    y = np.array([[[1.0]]])
    # y + b^2 * op * b^2 * x = 1 + 1.5^4 * 6
    assert oracle.mass_apply(y, B, op, x)[0, 0, 0] == 1.0 + 1.5 ** 4 * 6.0
