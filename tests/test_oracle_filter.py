"""Oracle pins for filtering on top of random-access decode:
closed-form special cases and the stochastic-filtering expectation."""
import numpy as np
import pytest

from paper_2305_17105_b200.synth import Profile
from helpers import material_inputs


@pytest.fixture(scope="module")
def mat(O):
    d = Profile.named("ntc0.2", 64, 4)
    codes, w = material_inputs(O, d, 17, out_gain=1.0)
    return d, codes, w


def test_bilinear_at_texel_centres_is_decode(O, mat):
    d, codes, w = mat
    rng = np.random.default_rng(0)
    q = []
    for _ in range(200):
        m = int(rng.integers(0, 7))
        wm = 64 >> m
        x, y = rng.integers(0, wm, 2)
        q.append((x, y, m))
    q = np.array(q, np.int32)
    uvl = np.stack([(q[:, 0] + 0.5) / (64 >> q[:, 2]), (q[:, 1] + 0.5) / (64 >> q[:, 2]), q[:, 2]], 1)
    ref = O.decode_texels(d, codes, w, q)
    assert np.array_equal(O.filter_texels(d, codes, w, uvl, 1), ref)
    assert np.array_equal(O.filter_texels(d, codes, w, uvl, 0), ref)
    assert np.array_equal(O.filter_texels(d, codes, w, uvl, 2), ref)  # integer LOD: one mip


def test_trilinear_blends_adjacent_mips(O, mat):
    d, codes, w = mat
    rng = np.random.default_rng(1)
    uv = rng.random((100, 2))
    for lod in (0.25, 1.5, 3.75):
        m = int(np.floor(lod))
        t = lod - m
        a = O.filter_texels(d, codes, w, np.c_[uv, np.full(100, m)], 1)
        b = O.filter_texels(d, codes, w, np.c_[uv, np.full(100, m + 1)], 1)
        got = O.filter_texels(d, codes, w, np.c_[uv, np.full(100, lod)], 2)
        assert np.allclose(got, (1 - t) * a + t * b, atol=1e-14)


@pytest.mark.parametrize("mode,ref_mode", [(3, 1), (4, 2)])
def test_stochastic_expectation(O, mat, mode, ref_mode):
    """U(-1/2,1/2) texel jitter + nearest decode has the bilinear filter as
    its expectation; with the LOD jittered too, the trilinear one.  Monte Carlo over 2e4
    independent samples per point, 4 sigma."""
    d, codes, w = mat
    rng = np.random.default_rng(2)
    pts = np.c_[rng.uniform(0.1, 0.9, (8, 2)), rng.uniform(0.2, 2.8, 8)]
    n = 20000
    for p in pts:
        uvl = np.repeat(p[None], n, 0)
        s = O.filter_texels(d, codes, w, uvl, mode, seed=7)
        want = O.filter_texels(d, codes, w, p[None], ref_mode)[0]
        se = s.std(0) / np.sqrt(n) + 1e-9
        assert np.all(np.abs(s.mean(0) - want) <= 4 * se + 1e-12), (p, s.mean(0), want)
