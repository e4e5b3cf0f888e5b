"""Pins for the batched multiply-accumulate oracle (§5.1, Listing 8).

The oracle computes c[b] += a[b] @ b[b] (reading R16).  Checked
against a hand-expanded example, exact rational arithmetic, and special cases
whose result is fixed exactly (identity / zero factors, transposition).
"""
from __future__ import annotations

import os
from fractions import Fraction

import numpy as np
import pytest

import jm_synth
import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _rows(s):
    return np.array([[float(v) for v in r.split()] for r in s.split(";")])


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_hand_expanded_2x2(dt):
    with open(os.path.join(GOLDEN, "mm_hand_2x2.txt")) as f:
        line = [ln for ln in f if ln.strip() and not ln.startswith("#")][0]
    a, b, c, want = (_rows(p).astype(dt)[None] for p in line.strip().split("|"))
    got = oracle.matmul_acc(c, a, b)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("n", [1, 2, 3, 5, 8])
def test_exact_rational_f64(n):
    a = jm_synth.generate(n, "f64", "bench", 1, 0, 4)
    b = jm_synth.generate(n, "f64", "bench", 2, 0, 4)
    c = jm_synth.generate(n, "f64", "bench", 3, 0, 4)
    got = oracle.matmul_acc(c, a, b)
    for bi in range(4):
        exact = [[Fraction(c[bi, i, j]) + sum(Fraction(a[bi, i, k]) * Fraction(b[bi, k, j])
                                              for k in range(n)) for j in range(n)] for i in range(n)]
        want = np.array([[float(v) for v in row] for row in exact])
        scale = np.max(np.abs(c[bi])) + np.max(np.sum(np.abs(a[bi])[:, :, None] * np.abs(b[bi])[None], axis=1))
        assert np.max(np.abs(got[bi] - want)) <= 2 * (n + 1) * np.finfo(np.float64).eps * scale


@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_identity_and_zero_factors_exact(dt):
    n = 6
    b = jm_synth.generate(n, dt, "bench", 4, 0, 3)
    c = jm_synth.generate(n, dt, "bench", 5, 0, 3)
    eye = np.broadcast_to(np.eye(n, dtype=b.dtype), b.shape).copy()
    assert np.array_equal(oracle.matmul_acc(c, eye, b), c + b)      # one rounding: c + b
    assert np.array_equal(oracle.matmul_acc(c, b, eye), c + b)
    assert np.array_equal(oracle.matmul_acc(c, np.zeros_like(b), b), c)


@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_transpose_bitwise(dt):
    n = 7
    a = jm_synth.generate(n, dt, "bench", 6, 0, 5)
    b = jm_synth.generate(n, dt, "bench", 7, 0, 5)
    c = jm_synth.generate(n, dt, "bench", 8, 0, 5)
    t = lambda x: np.ascontiguousarray(np.swapaxes(x, 1, 2))  # noqa: E731
    assert np.array_equal(oracle.matmul_acc(t(c), t(b), t(a)), t(oracle.matmul_acc(c, a, b)))


def test_batch_entries_independent_and_inputs_untouched():
    n = 4
    a = jm_synth.generate(n, "f64", "bench", 9, 0, 6)
    b = jm_synth.generate(n, "f64", "bench", 10, 0, 6)
    c = jm_synth.generate(n, "f64", "bench", 11, 0, 6)
    c0 = c.copy()
    whole = oracle.matmul_acc(c, a, b, threads=3)
    assert np.array_equal(c, c0)
    for i in range(6):
        assert np.array_equal(oracle.matmul_acc(c[i:i + 1], a[i:i + 1], b[i:i + 1], threads=1)[0], whole[i])


def test_transposed_operand_mutant_is_caught():
    n = 3
    a = jm_synth.generate(n, "f64", "bench", 12, 0, 1)
    b = jm_synth.generate(n, "f64", "bench", 13, 0, 1)
    c = np.zeros_like(a)
    good = oracle.matmul_acc(c, a, b)[0]
    assert not np.allclose(good, a[0].T @ b[0])
    assert not np.allclose(good, b[0] @ a[0])
