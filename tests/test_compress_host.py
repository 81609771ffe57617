"""CPU checks of the compression loop's host logic."""
import math

import numpy as np
import pytest

from paper_2305_17105_b200.compress import init_state, lr_at, sample_lod
from paper_2305_17105_b200.synth import Profile


def test_lod_law():
    """LOD = floor(-log4 X) -> P(k) = (3/4) 4^-k; P(0) in [0.747, 0.753] over
    10^6 draws."""
    rng = np.random.default_rng(0)
    n = 1_000_000
    draws = np.array([sample_lod(rng, 13, 0.0) for _ in range(n)])
    p = np.bincount(draws, minlength=13) / n
    assert 0.747 <= p[0] <= 0.753
    for k in range(1, 5):
        want = 0.75 * 4.0**-k
        assert abs(p[k] - want) < 4 * math.sqrt(want / n)


def test_lod_uniform_fraction_and_clamp():
    """5% of the batches are uniform over the chain; LODs clamp to M-1."""
    rng = np.random.default_rng(1)
    n = 400_000
    M = 3
    draws = np.array([sample_lod(rng, M, 0.05) for _ in range(n)])
    p = np.bincount(draws, minlength=M) / n
    want = [0.95 * 0.75 + 0.05 / 3, 0.95 * 0.1875 + 0.05 / 3, 0.95 * 0.0625 + 0.05 / 3]
    for k in range(M):
        assert abs(p[k] - want[k]) < 4 * math.sqrt(want[k] / n)
    assert draws.max() == M - 1


def test_cosine_schedule():
    """cosine annealing from the initial rate to 0."""
    assert lr_at(0, 1000, 0.01) == 0.01
    assert abs(lr_at(1000, 1000, 0.01)) < 1e-18
    assert abs(lr_at(500, 1000, 0.005) - 0.0025) < 1e-15
    assert all(lr_at(t, 100, 1.0) >= lr_at(t + 1, 100, 1.0) for t in range(100))


def test_init_state_in_range(O):
    d = Profile.named("ntc0.2", 64, 4)
    lat, par = init_state(d, 3, "cpu")
    lat = lat.numpy()
    for j in range(O.num_levels(d)):
        for k, B in ((0, d.b0), (1, d.b1)):
            a = O.grid_offset(d, j, k)
            b = O.grid_offset(d, j, 1) if k == 0 else O.grid_offset(d, j + 1, 0)
            lo, hi = O.quant_range(B)
            q = (hi - lo) / 4
            assert lat[a:b].min() >= lo + q - 1e-7 and lat[a:b].max() <= hi - q + 1e-7
    assert par.numel() == O.num_params(d)
