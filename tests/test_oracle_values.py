"""Oracle pins: quantisation, fp16 format, positional encoding, LOD, hardGELU, MLP,
Philox noise (CPU only).  Each check ties the oracle to the paper's stated property,
a closed form, a textbook/library routine, or brute force -- not to a retyped formula.
"""
import math

import numpy as np
import pytest
import torch

from conftest import golden
from paper_2305_17105_b200.synth import Profile, gen_weights_f16


# ---------------------------------------------------------------- quantisation
@pytest.mark.parametrize("B", range(1, 9))
def test_zero_is_a_bin_centre(O, B):
    """'This quantizes a zero value with no error'."""
    assert O.dequantize(O.quantize(0.0, B), B) == 0.0


@pytest.mark.parametrize("B", range(1, 9))
def test_range_and_centres(O, B):
    """range [-(N-1)/2 Q, N/2 Q], N = 2^B, Q = 1/N; N centres spaced Q."""
    N = 2**B
    lo, hi = O.quant_range(B)
    assert lo == -(N - 1) / 2 / N and hi == N / 2 / N
    centres = [O.dequantize(c, B) for c in range(N)]
    assert len(set(centres)) == N
    assert np.allclose(np.diff(centres), 1.0 / N, atol=0)
    assert centres[-1] == hi                      # top of the range is a centre
    assert centres[0] - lo == 0.5 / N             # bottom of the range is half a bin below
    for c in range(N):                            # quantize(dequantize(code)) = code
        assert O.quantize(centres[c], B) == c


@pytest.mark.parametrize("B", [1, 2, 3, 4, 8])
def test_quantize_brute_force_nearest(O, B):
    """Nearest centre by brute force over all N centres, ties to the larger centre (R9),
    for values across and beyond the range (clamped to the extreme centres)."""
    N = 2**B
    centres = np.array([O.dequantize(c, B) for c in range(N)])
    rng = np.random.default_rng(B)
    vals = np.concatenate([rng.uniform(-1.0, 1.0, 2000), centres + 0.5 / N, centres - 0.5 / N])
    for v in vals:
        dist = np.abs(centres - v)
        best = np.flatnonzero(dist == dist.min()).max()
        assert O.quantize(v, B) == best
        q = O.dequantize(O.quantize(v, B), B)
        assert O.quantize(q, B) == O.quantize(v, B)   # idempotent


def test_spec_quantize_clamp_examples(O):
    """SPEC.md:135-137, 153-155 (B = 2: centres -0.25, 0, 0.25, 0.5)."""
    assert O.dequantize(O.quantize(0.3, 2), 2) == 0.25
    assert O.dequantize(O.quantize(0.9, 2), 2) == 0.5
    lo, hi = O.quant_range(2)
    assert (lo, hi) == (-0.375, 0.5)
    assert O.dequantize(O.quantize(lo, 2), 2) == -0.25  # the tie at lo goes up (R9)


# ---------------------------------------------------------------- fp16 format
def test_f16_conversion_matches_numpy(O):
    """IEEE binary16 round-to-nearest-even vs numpy's float16 (library), incl. ties,
    subnormals and overflow."""
    rng = np.random.default_rng(0)
    v = np.concatenate([
        rng.normal(0, 1, 3000), rng.normal(0, 1e-5, 1000), rng.normal(0, 3e4, 500),
        np.array([0.0, -0.0, 65504.0, 65519.99, 65520.0, 2**-24, 2**-25, 3 * 2**-26, 2**-14, 1.0 + 2**-11,
                  1.0 + 3 * 2**-11, 0.1, 1 / 3]),
    ])
    for x in v:
        want = int(np.array(x).astype(np.float16).view(np.uint16))
        assert O.f64_to_f16(x) == want, x
    for h in range(0, 65536, 7):
        f = np.array(h, np.uint16).view(np.float16).astype(np.float64)
        if np.isnan(f):
            continue
        assert O.f16_to_f64(h) == f


def test_lod_fp16(O):
    """R6: LOD input = fp16(m / (M-1)); endpoints 0 and 1."""
    for W in (4, 256, 2048, 4096, 8192):
        M = O.num_mips(W)
        for m in range(M):
            want = int(np.array(m / (M - 1)).astype(np.float16).view(np.uint16))
            assert O.lod_f16(m, M) == want
        assert O.f16_to_f64(O.lod_f16(0, M)) == 0.0 and O.f16_to_f64(O.lod_f16(M - 1, M)) == 1.0


# ---------------------------------------------------------------- positional encoding
def test_triangle_wave_fourier(O):
    """tri(t) = (8/pi^2) sum_{k odd} cos(2 pi k t) / k^2 -- the Fourier series of the
    period-1 triangle wave with tri(0) = 1, tri(1/2) = -1 (textbook closed form)."""
    ks = np.arange(1, 40001, 2, dtype=np.float64)
    for t in np.linspace(-1.3, 2.1, 57):
        series = 8 / math.pi**2 * np.sum(np.cos(2 * math.pi * ks * t) / ks**2)
        assert abs(O.tri(t) - series) < 1e-4


def test_pe_table_golden(O):
    """The 8 x 6 per-axis PE table (tests/golden/pe_table.txt): it fixes
    the phase sign (+1/4 instead of -1/4 moves entries 2/4/6), the octave order and the
    integer (not texel-centre) position; the last column is the constant the Fig. 5 caption
    states.  Every (x, y) of a 16 x 16 patch: [PE_x(x mod 8) | PE_y(y mod 8)]."""
    from conftest import golden

    tab = {int(r[0]): np.array([float(v) for v in r[1:]]) for r in golden("pe_table.txt")}
    assert sorted(tab) == list(range(8))
    assert all(t[5] == 0.0 for t in tab.values())  # "the last value is constant"
    for y in range(16):
        for x in range(16):
            assert np.array_equal(O.pe(x, y), np.concatenate([tab[x % 8], tab[y % 8]])), (x, y)


def test_pe_properties(O):
    """PAPER.md:464 (tile repeats every 8x8), PAPER.md:468 ('6+6 scalars', 'the last value
    is constant in both the horizontal and vertical encoding')."""
    assert np.array_equal(O.pe(0, 0)[:6], [1, 0, 1, 0, 1, 0])
    seen_x = set()
    for x in range(-8, 24):
        for y in range(-8, 24, 5):
            p = O.pe(x, y)
            assert p.shape == (12,)
            assert np.array_equal(p, O.pe(x + 8, y)) and np.array_equal(p, O.pe(x, y + 8))
            assert p[5] == 0.0 and p[11] == 0.0             # last value constant
            assert np.all(np.abs(p) <= 1.0)
            assert np.array_equal(p[:6], O.pe(x, 0)[:6])     # x half depends on x only
            seen_x.add(tuple(p[:6]))
    assert len(seen_x) == 8   # distinct code for every position in the tile


def test_pe_octaves(O):
    """3 octaves = log2 8: octave h has period 8 / 2^h texels."""
    for x in range(8):
        p = O.pe(x, 0)
        for h, period in enumerate((8, 4, 2)):
            assert p[2 * h] == O.pe(x + period, 0)[2 * h]


# ---------------------------------------------------------------- hardGELU
def test_hardgelu_paper_values(O):
    """PAPER.md:498-504 piecewise definition; SPEC.md:198-201 examples; continuity."""
    assert O.hardgelu(-2.0) == 0.0
    assert O.hardgelu(2.0) == 2.0
    assert O.hardgelu(0.0) == 0.0
    assert O.hardgelu(1.5) == 1.5 and O.hardgelu(-1.5) == 0.0
    for k in (-1.5, 1.5):
        assert abs(O.hardgelu(k - 1e-9) - O.hardgelu(k + 1e-9)) < 1e-8


def test_hardgelu_is_scaled_hardswish(O):
    """'similar to hard Swish': hardGELU(x) = hardswish(2x)/2, with torch's
    hardswish (x * relu6(x+3)/6) as the library routine."""
    xs = torch.linspace(-5, 5, 2001, dtype=torch.float64)
    ref = torch.nn.functional.hardswish(2 * xs) / 2
    got = torch.tensor([O.hardgelu(float(x)) for x in xs], dtype=torch.float64)
    assert torch.allclose(got, ref, atol=1e-15, rtol=0)


def test_hardgelu_vs_gelu(O):
    """max |hardGELU - GELU| on [-4, 4] (SPEC.md:218 bound 0.2; SURVEY computed 0.1002)."""
    xs = np.arange(-4.0, 4.0 + 1e-12, 1e-3)
    gelu = np.array([x * 0.5 * (1 + math.erf(x / math.sqrt(2))) for x in xs])
    hg = np.array([O.hardgelu(x) for x in xs])
    err = np.max(np.abs(hg - gelu))
    assert err < 0.2
    assert abs(err - 0.1002) < 5e-4


def test_hardgelu_grad_finite_difference(O):
    """R15: derivative = central differences away from the kinks, middle slope at them."""
    h = 1e-6
    for x in np.linspace(-3, 3, 301):
        if min(abs(x - 1.5), abs(x + 1.5)) < 1e-3:
            continue
        fd = (O.hardgelu(x + h) - O.hardgelu(x - h)) / (2 * h)
        assert abs(fd - O.hardgelu_grad(x)) < 1e-6
    assert O.hardgelu_grad(1.5) == 1.5 and O.hardgelu_grad(-1.5) == -0.5


# ---------------------------------------------------------------- exact GELU (f4)
def test_gelu_matches_torch(O):
    """activation = 1 is GELU: torch's exact (erf) GELU and its autograd
    derivative as the library routines."""
    xs = torch.linspace(-6, 6, 2401, dtype=torch.float64, requires_grad=True)
    ref = torch.nn.functional.gelu(xs, approximate="none")
    (gref,) = torch.autograd.grad(ref.sum(), xs)
    got = np.array([O.gelu(float(x)) for x in xs.detach()])
    gg = np.array([O.gelu_grad(float(x)) for x in xs.detach()])
    assert np.allclose(got, ref.detach().numpy(), atol=1e-14, rtol=0)
    assert np.allclose(gg, gref.numpy(), atol=1e-13, rtol=0)


def test_gelu_identities(O):
    """x Phi(x) closed forms: GELU(0) = 0, GELU(x) - GELU(-x) = x (Phi(x) + Phi(-x) = 1),
    GELU'(0) = 1/2, GELU'(x) + GELU'(-x) = 1, and GELU(x) -> x / 0 in the tails."""
    assert O.gelu(0.0) == 0.0 and O.gelu_grad(0.0) == 0.5
    for x in np.linspace(-5, 5, 101):
        assert abs(O.gelu(x) - O.gelu(-x) - x) < 1e-14
        assert abs(O.gelu_grad(x) + O.gelu_grad(-x) - 1.0) < 1e-14
    assert abs(O.gelu(12.0) - 12.0) < 1e-15 and abs(O.gelu(-12.0)) < 1e-15
    h = 1e-6
    for x in np.linspace(-4, 4, 81):
        assert abs((O.gelu(x + h) - O.gelu(x - h)) / (2 * h) - O.gelu_grad(x)) < 1e-8


# ---------------------------------------------------------------- MLP
@pytest.mark.parametrize("hidden_mats,c,act", [(1, 8, 0), (1, 16, 0), (2, 9, 0), (1, 9, 1), (2, 8, 1)])
def test_mlp_matches_torch(O, hidden_mats, c, act):
    """Reduces to library routines: torch fp64 Linear layers + hardswish(2x)/2 (activation 0)
    or exact GELU (activation 1), no output activation."""
    d = Profile.named("ntc0.2", 64, c, hidden_mats, act)
    D = d.input_dim
    w = gen_weights_f16(11, D, c, hidden_mats).view(np.float16).astype(np.float64)
    rng = np.random.default_rng(1)
    X = rng.uniform(-1, 1, size=(50, D))
    dims = [(D, 64)] + [(64, 64)] * hidden_mats + [(64, c)]
    layers, off = [], 0
    for fi, fo in dims:
        lin = torch.nn.Linear(fi, fo).double()
        with torch.no_grad():
            lin.weight.copy_(torch.tensor(w[off: off + fi * fo].reshape(fo, fi)))
            off += fi * fo
            lin.bias.copy_(torch.tensor(w[off: off + fo]))
            off += fo
        layers.append(lin)
    assert off == O.num_params(d)
    with torch.no_grad():
        h = torch.tensor(X)
        for i, lin in enumerate(layers):
            h = lin(h)
            if i < len(layers) - 1:
                h = torch.nn.functional.hardswish(2 * h) / 2 if act == 0 else torch.nn.functional.gelu(h)
    for i in range(X.shape[0]):
        y = O.mlp_forward(d, w, X[i])
        assert np.allclose(y, h[i].numpy(), atol=1e-12, rtol=0)


def test_mlp_zero_weights_gives_bias(O):
    """all-zero weights -> output = output bias."""
    d = Profile.named("ntc0.2", 64, 9)
    P = O.num_params(d)
    w = np.zeros(P)
    w[-9:] = np.arange(9) * 0.1
    assert np.allclose(O.mlp_forward(d, w, np.random.default_rng(0).normal(size=57)), np.arange(9) * 0.1,
                       atol=0)


def test_param_count(O):
    """8,457 parameters for NTC 0.2, c = 9, [57, 64, 64, 9]."""
    assert O.num_params(Profile.named("ntc0.2", 4096, 9)) == 8457


# ---------------------------------------------------------------- Philox noise
def test_philox_known_answers(O):
    """Random123 known-answer vectors (tests/golden/philox_kat.txt)."""
    for row in golden("philox_kat.txt"):
        v = [int(t, 16) for t in row]
        assert O.philox(v[0:4], v[4:6]).tolist() == v[6:10]


@pytest.mark.parametrize("B", [2, 4])
def test_noise_distribution(O, B):
    """U(-Q/2, Q/2); support strictly inside, mean 0 and variance Q^2/12
    within 4 sigma."""
    Q = 1.0 / 2**B
    n = 100_000
    v = np.array([O.noise(0x1234, 7, i, B) for i in range(n)])
    assert np.all(v > -Q / 2) and np.all(v < Q / 2)
    sd = Q / math.sqrt(12)
    assert abs(v.mean()) < 4 * sd / math.sqrt(n)
    assert abs(v.var() - Q * Q / 12) < 4 * (Q * Q / math.sqrt(180)) / math.sqrt(n)
    # exact in fp32 (odd multiples of 2^-24 Q)
    assert np.array_equal(v.astype(np.float32).astype(np.float64), v)
    # one draw per latent per step: different steps give different values
    assert O.noise(0x1234, 8, 5, B) != O.noise(0x1234, 7, 5, B)
