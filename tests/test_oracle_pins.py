"""Pins for the CPU oracle.

Each test checks the oracle against something other than itself: a value the
paper/SPEC prints, a closed form, an invariant, exact rational brute force, or
a special case that reduces to a scalar recurrence.  A plausible mistake in the
oracle (dropped term, wrong sign/index, transposed operand, wrong constant,
in-place update instead of simultaneous) fails at least one of them — see
test_pins_catch_mutants at the bottom, which re-derives each mutant in plain
numpy and asserts that some pin rejects it.
"""
from __future__ import annotations

import os
from decimal import Decimal, getcontext
from fractions import Fraction

import numpy as np
import pytest

import jm_synth
import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
C64 = float(np.float64(0.00005))
C32 = float(np.float32(0.00005))


def _np(dt):
    return np.float64 if dt == "f64" else np.float32


def _golden_lines(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return [ln.split() for ln in f if ln.strip() and not ln.startswith("#")]


def _parse_rows(tokens):
    rows = " ".join(tokens).split(";")
    return np.array([[float(v) for v in r.split()] for r in rows], dtype=np.float64)


# ---------------------------------------------------------------- O1, O2, O3
def test_o1_spec_worked_example():
    for n, dt, addend, rep, x, want in _golden_lines("o1_spec_worked_example.txt"):
        inp = np.full((1, int(n), int(n)), float(x), dtype=_np(dt))
        out = oracle.run(inp, int(rep), addend)
        assert out.dtype == _np(dt)
        assert out[0, 0, 0] == _np(dt)(float(want))


def test_o2_initial_fill_matches_listing():
    for toks in _golden_lines("o2_initial_fill.txt"):
        n = int(toks[0])
        want = _parse_rows(toks[1:])
        buf = jm_synth.generate(n, "f64", "paper", 0, 0, 1).reshape(-1)
        # Eigen is column-major: m(i,j) = buf[i + n*j]
        m = buf.reshape(n, n).T
        np.testing.assert_array_equal(m, want)


def test_o3_hand_expanded_step():
    buf = jm_synth.generate(2, "f64", "paper", 0, 0, 1)
    for toks in _golden_lines("o3_hand_step_n2.txt"):
        addend, want = toks[0], _parse_rows(toks[1:])
        out = oracle.run(buf, 1, addend)[0]
        got = out.reshape(-1).reshape(2, 2).T  # back to m(i,j) column-major view
        assert np.array_equal(got, want), (addend, got, want)


# ---------------------------------------------------------------- O4, O5 fixed points
def _astar(n: int, c: float, digits: int = 60) -> Decimal:
    """Root of c*n*a^2 + (c-1)*a + 1 = 0 near 1 (stable form)."""
    getcontext().prec = digits
    c = Decimal(c)
    one = Decimal(1)
    return 2 / ((one - c) + ((one - c) ** 2 - 4 * c * n).sqrt())


def _xstar(c: float, digits: int = 60) -> Decimal:
    """Identity-variant fixed point x = 1 + c(x + x^2)."""
    getcontext().prec = digits
    c = Decimal(c)
    one = Decimal(1)
    return 2 / ((one - c) + ((one - c) ** 2 - 4 * c).sqrt())


def _ulps(a: np.ndarray, b: float, dt) -> float:
    eps = np.finfo(dt).eps
    return float(np.max(np.abs(a.astype(np.float64) - b)) / (abs(b) * eps))


def test_o4_c1_expected_output_paper_init():
    # BASELINE.json configs[0]: single FP64 4x4, paper's recurrence, 1000 repeats.
    x = jm_synth.generate(4, "f64", "paper", 0, 0, 1)
    out = oracle.run(x, 1000)
    a = float(_astar(4, C64))
    assert a == 1.0002501125631647  # value recorded in BASELINE.md §3
    assert _ulps(out, a, np.float64) <= 2.0


@pytest.mark.parametrize("n", [2, 3, 8, 16, 32])
def test_o4_fixed_point_f64(n):
    x = jm_synth.generate(n, "f64", "paper", 0, 0, 1)
    out = oracle.run(x, 150)
    assert _ulps(out, float(_astar(n, C64)), np.float64) <= 4.0


@pytest.mark.parametrize("n", [2, 4, 8, 16])
def test_o4_fixed_point_f32(n):
    x = jm_synth.generate(n, "f32", "bench", jm_synth.SEED_BENCH, 0, 2)
    out = oracle.run(x, 150)
    a = np.float32(float(_astar(n, C32)))
    assert out.dtype == np.float32
    assert _ulps(out, float(a), np.float32) <= 4.0 * n


def test_o5_identity_fixed_point():
    x = jm_synth.generate(4, "f64", "paper", 0, 0, 1)
    out = oracle.run(x, 1000, "identity")[0]
    xs = float(_xstar(C64))
    assert xs == pytest.approx(1.0001000150027506, abs=0, rel=2e-16)
    d = np.diag(out)
    assert _ulps(d, xs, np.float64) <= 2.0
    off = out - np.diag(d)
    assert np.all(off == 0.0)


# ---------------------------------------------------------------- O6 span{I,J}
@pytest.mark.parametrize("n,alpha,beta", [(3, 0.5, 2.0), (5, -0.25, 7.0), (8, 0.0, 3.0), (16, 1.5, -0.5)])
def test_o6_two_parameter_family_ones(n, alpha, beta):
    c = Fraction(C64)
    a, b = Fraction(alpha), Fraction(beta)
    m = (alpha * np.ones((n, n)) + beta * np.eye(n))[None]
    for r in range(1, 5):
        a, b = 1 + c * (a + n * a * a + 2 * a * b), c * (b + b * b)
        a = Fraction(float(a)); b = Fraction(float(b))  # keep sizes small
        want = float(a) * np.ones((n, n)) + float(b) * np.eye(n)
        got = oracle.run(m, r)[0]
        err = np.max(np.abs(got - want)) / np.max(np.abs(want))
        assert err < 1e-14, (r, err)


# ---------------------------------------------------------------- O7 row sums
@pytest.mark.parametrize("n", [3, 6, 11])
def test_o7_row_sum_invariant(n):
    rng = np.random.default_rng(7 + n)
    m = rng.uniform(-1, 1, (n, n))
    sigma = 2.5
    m += (sigma - m.sum(axis=1, keepdims=True)) / n  # every row sums to sigma
    s = Fraction(sigma)
    c = Fraction(C64)
    for r in range(1, 5):
        s = n + c * (s + s * s)
        got = oracle.run(m[None], r)[0]
        np.testing.assert_allclose(got.sum(axis=1), float(s), rtol=1e-13)


def test_o7_nilpotent_zero_sum_ones():
    # N = u v^T with 1^T u = v^T 1 = v^T u = 0  =>  N^2 = 0, N 1 = 0, 1^T N = 0.
    u = np.array([1.0, -1.0, 2.0, -2.0])
    v = np.array([1.0, 1.0, -1.0, -1.0])
    assert u.sum() == 0 and v.sum() == 0 and v @ u == 0
    N = np.outer(u, v)
    n = 4
    c = Fraction(C64)
    a = Fraction(0)
    for k in range(1, 5):
        a = 1 + c * (a + n * a * a)
        want = float(a) * np.ones((n, n)) + float(c ** k) * N
        got = oracle.run(N[None], k)[0]
        np.testing.assert_allclose(got, want, rtol=1e-14, atol=1e-300)


# ---------------------------------------------------------------- O8 identity-variant forms
@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_o8_scalar_identity_and_diagonal_bitwise(dt):
    T = _np(dt)
    c = T(0.00005)
    d0 = np.array([0.0, 0.5, -0.75, 3.0, 100.0], dtype=T)
    m = np.diag(d0)[None]
    x = d0.copy()
    for r in range(1, 6):
        x = (T(1) + c * (x + x * x)).astype(T)   # elementwise scalar recurrence
        got = oracle.run(m, r, "identity")[0]
        assert np.array_equal(np.diag(got), x)
        assert np.all(got[~np.eye(5, dtype=bool)] == 0)


def test_o8_nilpotent_identity_variant():
    n = 4
    N = np.triu(np.ones((n, n)), 3)  # single nonzero at (0,3): N^2 = 0
    s0, t0 = 0.3, 5.0
    m = s0 * np.eye(n) + t0 * N
    c = Fraction(C64)
    x, y = Fraction(s0), Fraction(t0)
    for k in range(1, 5):
        x, y = 1 + c * (x + x * x), c * y * (1 + 2 * x)
        want = float(x) * np.eye(n) + float(y) * N
        got = oracle.run(m[None], k, "identity")[0]
        np.testing.assert_allclose(got, want, rtol=1e-14, atol=0)


def test_o8_strictly_upper_stays_upper():
    n = 6
    rng = np.random.default_rng(3)
    m = np.triu(rng.uniform(-2, 2, (n, n)), 1)
    for r in (1, 2, 5):
        got = oracle.run(m[None], r, "identity")[0]
        assert np.all(np.tril(got, -1) == 0)
        x = 0.0
        for _ in range(r):
            x = 1.0 + C64 * (x + x * x)
        assert np.all(np.diag(got) == x)


# ---------------------------------------------------------------- O9 equivariance
@pytest.mark.parametrize("dt", ["f64", "f32"])
@pytest.mark.parametrize("addend", ["ones", "identity"])
def test_o9_transpose_equivariance_bitwise(dt, addend):
    n = 7
    x = jm_synth.generate(n, dt, "hard", jm_synth.SEED_HARD_BASE + n, 0, 8)
    a = oracle.run(x, 3, addend)
    b = oracle.run(np.ascontiguousarray(np.swapaxes(x, 1, 2)), 3, addend)
    assert np.array_equal(np.swapaxes(b, 1, 2), a)


# ---------------------------------------------------------------- O10 exact brute force
def _exact_steps(m, reps, c, identity=False):
    n = len(m)
    F = [[Fraction(v) for v in row] for row in m]
    for _ in range(reps):
        P = [[sum(F[i][k] * F[k][j] for k in range(n)) for j in range(n)] for i in range(n)]
        F = [[(1 if (not identity or i == j) else 0) + c * (F[i][j] + P[i][j])
              for j in range(n)] for i in range(n)]
    return np.array([[float(v) for v in row] for row in F])


@pytest.mark.parametrize("n", [1, 2, 3, 4])
@pytest.mark.parametrize("addend", ["ones", "identity"])
def test_o10_exact_rational_bruteforce_f64(n, addend):
    x = jm_synth.generate(n, "f64", "hard", jm_synth.SEED_HARD_BASE + n, 0, 3)
    for reps in (1, 2, 3):
        got = oracle.run(x, reps, addend)
        for b in range(x.shape[0]):
            want = _exact_steps(x[b], reps, Fraction(C64), addend == "identity")
            err = np.max(np.abs(got[b] - want)) / np.max(np.abs(want))
            assert err <= 8 * n * reps * np.finfo(np.float64).eps, (reps, b, err)


def test_o10_hand_expanded_2x2_product():
    # [[a b],[c d]]^2 = [[a^2+bc, ab+bd],[ca+dc, cb+d^2]]; one Ones step in Fractions
    a, b, c_, d = 1.25, -0.5, 3.0, 0.75
    m = np.array([[a, b], [c_, d]])
    sq = np.array([[a * a + b * c_, a * b + b * d], [c_ * a + d * c_, c_ * b + d * d]])
    want = np.array([[float(1 + Fraction(C64) * (Fraction(m[i, j]) + Fraction(sq[i, j])))
                      for j in range(2)] for i in range(2)])
    got = oracle.run(m[None], 1)[0]
    np.testing.assert_allclose(got, want, rtol=2e-16, atol=0)


@pytest.mark.parametrize("n", [2, 3])
def test_o10_exact_rational_bruteforce_f32(n):
    x = jm_synth.generate(n, "f32", "hard", jm_synth.SEED_HARD_BASE + n, 0, 2)
    got = oracle.run(x, 2)
    for b in range(2):
        want = _exact_steps(x[b].astype(np.float64), 2, Fraction(C32))
        err = np.max(np.abs(got[b] - want)) / np.max(np.abs(want))
        assert err <= 8 * n * 2 * np.finfo(np.float32).eps


# ---------------------------------------------------------------- O11
@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_o11_repeat_zero_is_copy_and_batch_independence(dt):
    n = 5
    x = jm_synth.generate(n, dt, "bench", jm_synth.SEED_BENCH, 0, 9)
    assert np.array_equal(oracle.run(x, 0), x)
    whole = oracle.run(x, 4, threads=3)
    for b in range(9):
        assert np.array_equal(oracle.run(x[b:b + 1], 4, threads=1)[0], whole[b])
    # slicing the generator by global index gives the same inputs (W-invariance)
    part = jm_synth.generate(n, dt, "bench", jm_synth.SEED_BENCH, 4, 5)
    assert np.array_equal(part, x[4:])


# ---------------------------------------------------------------- O12 divergence
@pytest.mark.parametrize("n,rep", [(35, 14), (40, 11), (48, 10), (64, 9)])
def test_o12_paper_init_diverges_to_inf(n, rep):
    x = jm_synth.generate(n, "f64", "paper", 0, 0, 1)
    out = oracle.run(x, rep)
    assert np.all(np.isposinf(out))


def test_o12_n34_stays_finite():
    x = jm_synth.generate(34, "f64", "paper", 0, 0, 1)
    out = oracle.run(x, 199)
    assert np.all(np.isfinite(out))
    assert _ulps(out, float(_astar(34, C64)), np.float64) <= 8.0


# ---------------------------------------------------------------- generator pins
def test_generator_splitmix_reference_vector():
    # splitmix64 with state 0: first output is 0xE220A8397B1DCDAF (Vigna).
    z = jm_synth.splitmix64_finalize(np.array([0x9E3779B97F4A7C15], dtype=np.uint64))
    assert int(z[0]) == 0xE220A8397B1DCDAF
    u = jm_synth.uniform01(0, 1, 0, 1)
    assert u[0] == (0xE220A8397B1DCDAF >> 11) * 2.0 ** -53


def test_constants():
    assert C32 == 4.999999873689376e-05
    assert C64 == 5.0000000000000002e-05


# ---------------------------------------------------------------- the pins bite
def _mutant_step(m, kind):
    n = m.shape[0]
    c = 0.00005
    if kind == "transposed":
        p = m.T @ m
    elif kind == "dropped_k":
        p = m[:, 1:] @ m[1:, :]
    elif kind == "no_m_term":
        return 1.0 + c * (m @ m)
    elif kind == "sign":
        p = -(m @ m)
    elif kind == "identity_as_ones":
        return np.eye(n) + c * (m + m @ m)
    elif kind == "c_float":
        return 1.0 + float(np.float32(c)) * (m + m @ m)
    elif kind == "inplace":
        m = m.copy()
        for i in range(n):
            for j in range(n):
                m[i, j] = 1.0 + c * (m[i, j] + m[i, :] @ m[:, j])
        return m
    return 1.0 + c * (m + p)


@pytest.mark.parametrize("kind", ["transposed", "dropped_k", "no_m_term", "sign",
                                  "identity_as_ones", "c_float", "inplace"])
def test_pins_catch_mutants(kind):
    """A mutated update must violate O3 or O10 (so those pins can detect it)."""
    x = jm_synth.generate(3, "f64", "hard", jm_synth.SEED_HARD_BASE + 3, 0, 1)[0]
    want = _exact_steps(x, 1, Fraction(C64))
    bad = _mutant_step(x, kind)
    err = np.max(np.abs(bad - want)) / np.max(np.abs(want))
    buf = jm_synth.generate(2, "f64", "paper", 0, 0, 1)[0]
    o3 = np.array([[1.0001, 1.0002], [1.0004, 1.0007]])
    o3_bad = not np.array_equal(_mutant_step(buf, kind), o3)
    assert err > 24 * np.finfo(np.float64).eps or o3_bad
