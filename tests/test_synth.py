"""The seeded input generator (jm_synth): ranges, signs and batch-slice
invariance of every distribution, including the signed parity-hard one."""
from __future__ import annotations

import numpy as np
import pytest

import jm_synth


@pytest.mark.parametrize("dt", ["f32", "f64"])
@pytest.mark.parametrize("n", [1, 7, 16, 33, 64])
def test_ranges_and_signs(n, dt):
    h = jm_synth.generate(n, dt, "hard", 5, 0, 50)
    s = jm_synth.generate(n, dt, "shard", 5, 0, 50)
    b = jm_synth.generate(n, dt, "bench", 5, 0, 50)
    lim = 2 * jm_synth.RHO_HARD / n
    assert h.min() >= 0 and h.max() < lim * (1 + 1e-6)
    assert s.min() >= -lim * (1 + 1e-6) and s.max() < lim * (1 + 1e-6)
    assert b.min() >= -1 and b.max() < 1
    if n * n * 50 >= 1000:                      # both signs present in bulk
        assert (s < 0).mean() > 0.4 and (s > 0).mean() > 0.4
    # same counter stream: shard = 2*hard - lim up to rounding
    np.testing.assert_allclose(s.astype(np.float64), (2 * h.astype(np.float64) - lim), rtol=0, atol=lim * 1e-6)


@pytest.mark.parametrize("dist", ["paper", "bench", "hard", "shard"])
def test_slices_equal_whole_batch(dist):
    whole = jm_synth.generate(9, "f64", dist, 123, 0, 40)
    parts = np.concatenate([jm_synth.generate(9, "f64", dist, 123, a, b - a) for a, b in ((0, 13), (13, 29), (29, 40))])
    assert np.array_equal(whole.view(np.uint64), parts.view(np.uint64))
