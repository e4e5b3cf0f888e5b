"""Seeded synthetic inputs for the batched Eigen-benchmark update (host side).

This module is shared by the tests, ``bench.py`` and the oracle harness.  It
holds NONE of the method's arithmetic (no matrix product, no update): only

* the counter-based input generator (SURVEY.md §8(d) "Input generator"),
  keyed by the GLOBAL matrix index so that a batch sliced across W ranks is
  bit-identical to the unsliced batch ("a proxy for part of a
  larger computation");
* the input distributions ``paper`` / ``bench`` / ``hard`` / ``shard``;
* the order-independent u64 checksum used by the multi-GPU gather (plumbing,
  SURVEY.md §8(e)); the device re-implements both (csrc/kernels/jm_aux.cuh) —
  the two sides share no code, only this written definition:

    z = seed ^ (0x9E3779B97F4A7C15 * (g*n*n + e + 1))        (mod 2^64)
    z = splitmix64_finalize(z)
    u = (z >> 11) * 2^-53                                     (U[0,1), double)

    paper : x = e                    (iota; = i + n*j read column-major,
                                      PAPER.md:374-377 Listing 4)
    bench : x = T(2u - 1)            (U[-1,1), throughput runs)
    hard  : x = T(u * 2*rho/n)       (rho = 4000: c*rho = 0.2, parity-hard)
    shard : x = T((2u - 1) * 2*rho/n) (signed parity-hard: cancellation in M*M,
                                      sign errors visible)

    checksum: S = sum_e mix64(bits(x_e) ^ (PHI * (g*n*n + e)))   (mod 2^64)
              with bits() the IEEE bit pattern zero-extended to 64 bits.
"""
from __future__ import annotations

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
PHI = np.uint64(0x9E3779B97F4A7C15)
RHO_HARD = 4000.0

DIST_PAPER = 0
DIST_BENCH = 1
DIST_HARD = 2
DIST_SHARD = 3
DISTS = {"paper": DIST_PAPER, "bench": DIST_BENCH, "hard": DIST_HARD, "shard": DIST_SHARD}

SEED_BENCH = 0x0019040855
SEED_HARD_BASE = 0x5EED0000

_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64_finalize(z: np.ndarray) -> np.ndarray:
    """Standard splitmix64 output mixer on a uint64 array (wrapping)."""
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = z ^ (z >> np.uint64(30))
        z = z * _M1
        z = z ^ (z >> np.uint64(27))
        z = z * _M2
        z = z ^ (z >> np.uint64(31))
    return z


def _np_dtype(dtype) -> np.dtype:
    if dtype in ("f32", "float", np.float32, 0):
        return np.dtype(np.float32)
    if dtype in ("f64", "double", np.float64, 1):
        return np.dtype(np.float64)
    raise ValueError(f"unsupported dtype {dtype!r}")


def uniform01(seed: int, n: int, global_first: int, batch: int) -> np.ndarray:
    """U[0,1) doubles for matrices [global_first, global_first+batch), flat."""
    nn = n * n
    idx = np.arange(global_first * nn, (global_first + batch) * nn, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed) ^ (GOLDEN * (idx + np.uint64(1)))
    z = splitmix64_finalize(z)
    return (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def generate(n: int, dtype, dist: str | int, seed: int, global_first: int = 0,
             batch: int = 1) -> np.ndarray:
    """Return a (batch, n, n) array of the requested distribution.

    The flat buffer is what the C ABI sees: matrix b occupies elements
    [b*n*n, (b+1)*n*n).  Viewing it as (batch, n, n) row-major is one of the two
    valid storage readings.
    """
    dt = _np_dtype(dtype)
    d = DISTS[dist] if isinstance(dist, str) else int(dist)
    nn = n * n
    if batch == 0:
        return np.zeros((0, n, n), dtype=dt)
    if d == DIST_PAPER:
        x = np.tile(np.arange(nn, dtype=np.float64), batch)
    else:
        u = uniform01(seed, n, global_first, batch)
        if d == DIST_BENCH:
            x = 2.0 * u - 1.0
        elif d == DIST_HARD:
            x = u * (2.0 * RHO_HARD / n)
        elif d == DIST_SHARD:
            x = (2.0 * u - 1.0) * (2.0 * RHO_HARD / n)
        else:
            raise ValueError(f"unknown dist {dist!r}")
    return x.astype(dt).reshape(batch, n, n)


def generate_chunked(n: int, dtype, dist, seed: int, global_first: int, batch: int,
                     out: np.ndarray | None = None, chunk: int = 1 << 16) -> np.ndarray:
    """Same as :func:`generate` but bounded temporaries (large host batches)."""
    dt = _np_dtype(dtype)
    if out is None:
        out = np.empty((batch, n, n), dtype=dt)
    for b0 in range(0, batch, chunk):
        b1 = min(batch, b0 + chunk)
        out[b0:b1] = generate(n, dt, dist, seed, global_first + b0, b1 - b0)
    return out


def checksum(x: np.ndarray, n: int, global_first: int = 0) -> int:
    """Order-independent u64 checksum of a flat batch (see module doc)."""
    x = np.ascontiguousarray(x)
    if x.dtype == np.float64:
        bits = x.reshape(-1).view(np.uint64)
    elif x.dtype == np.float32:
        bits = x.reshape(-1).view(np.uint32).astype(np.uint64)
    else:
        raise ValueError("checksum expects float32/float64")
    e = np.arange(global_first * n * n, global_first * n * n + bits.size, dtype=np.uint64)
    with np.errstate(over="ignore"):
        h = splitmix64_finalize(bits ^ (PHI * e))
        s = np.sum(h, dtype=np.uint64)
    return int(s)
