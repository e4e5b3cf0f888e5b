"""Parity metric shared by the GPU tests (SURVEY.md §8(c) "Parity protocol").

Per matrix b:  e_b = max_ij |G - O| / max_ij |O| over the finite entries, and
non-finite entries must agree position-wise (both NaN, or the same infinity).
Tolerances are the north star's: FP64 1e-12, FP32 1e-5 (BASELINE.json).
"""
from __future__ import annotations

import numpy as np

TOL = {np.dtype(np.float64): 1e-12, np.dtype(np.float32): 1e-5}


def max_rel_err(got: np.ndarray, want: np.ndarray) -> float:
    got = np.asarray(got)
    want = np.asarray(want)
    assert got.shape == want.shape, (got.shape, want.shape)
    if got.size == 0:
        return 0.0
    fin_w = np.isfinite(want)
    fin_g = np.isfinite(got)
    if not np.array_equal(fin_w, fin_g):
        return float("inf")
    nf = ~fin_w
    if nf.any():
        gw, ww = got[nf], want[nf]
        if not (np.array_equal(np.isnan(gw), np.isnan(ww))
                and np.array_equal(gw[~np.isnan(gw)], ww[~np.isnan(ww)])):
            return float("inf")
    g = np.where(fin_w, got, 0).astype(np.float64).reshape(got.shape[0], -1)
    w = np.where(fin_w, want, 0).astype(np.float64).reshape(want.shape[0], -1)
    den = np.max(np.abs(w), axis=1)
    num = np.max(np.abs(g - w), axis=1)
    den = np.where(den == 0, 1.0, den)
    return float(np.max(num / den))


def assert_parity(got, want, tol=None, what=""):
    tol = TOL[np.asarray(want).dtype] if tol is None else tol
    err = max_rel_err(got, want)
    assert err <= tol, f"{what}: max normwise rel err {err:.3e} > {tol:.1e}"
    return err
