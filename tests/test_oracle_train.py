"""Oracle pins for the training step and decode composition (CPU only).

- gradients: central finite differences in fp64 on tiny materials;
- Adam: torch.optim.Adam (library routine) and the closed-form first step;
- invariants: channel-permutation symmetry, clamp-after-update;
- decode composition: an independent decode built from library routines (grid_sample,
  torch Linear, hardswish, the triangle-wave Fourier series) equals the oracle decode.
"""
import math

import numpy as np
import pytest
import torch

from paper_2305_17105_b200.synth import (Profile, box_mip_chain_u8, gen_codes, gen_crops, gen_latents,
                                         gen_reference_u8, gen_weights_f16, gen_weights_f32, u8_to_f16_bits)


def _material(O, d, seed):
    lat = gen_latents(seed, O.num_latents(d))
    par = gen_weights_f32(seed + 1, d.input_dim, d.channels, d.hidden_mats, out_gain=1.0)
    chain = box_mip_chain_u8(gen_reference_u8(seed + 2, d.width, d.channels))
    return lat, par, chain


@pytest.mark.parametrize("mip,hidden,act,profile", [(0, 1, 0, "ntc0.2"), (1, 1, 0, "ntc0.2"), (4, 1, 0, "ntc0.2"),
                                                    (0, 2, 0, "ntc0.2"), (0, 1, 1, "ntc0.2"), (1, 2, 1, "ntc0.2"),
                                                    (0, 1, 0, "ntc2.25"), (1, 1, 0, "ntc1.0")])
def test_gradients_finite_difference(O, mip, hidden, act, profile):
    """Analytic gradients vs central differences (exact-input mode, h = 1e-6): per-tensor
    relative L2 error < 1e-4 on sampled weights and every touched latent sample; hardGELU
    (act 0) and exact GELU (act 1, the f4 variant)."""
    d = Profile.named(profile, 32, 3, hidden, act)
    lat, par, chain = _material(O, d, 100 + mip)
    ref = u8_to_f16_bits(chain[mip])
    crops = gen_crops(5, 32, mip, 2, crop=8)
    args = dict(mip=mip, crops=crops, ref_f16=ref, seed=99, step=3, noise_on=True, round_f16=False)
    loss, dp, dl = O.train_grads(d, lat, par, **args)
    rng = np.random.default_rng(mip)
    h = 1e-6

    def L(l, p):
        # parameters are fp32: the divisor below is the representable perturbation actually made
        return O.train_grads(d, l, p, **args)[0]

    # weights
    idx = rng.choice(par.size, 200, replace=False)
    fd, an = [], []
    for i in idx:
        pp, pm = par.copy(), par.copy()
        pp[i] = np.float32(par[i] + h * max(1.0, abs(par[i])))
        pm[i] = np.float32(par[i] - h * max(1.0, abs(par[i])))
        dlt = float(pp[i]) - float(pm[i])
        fd.append((L(lat, pp) - L(lat, pm)) / dlt)
        an.append(dp[i])
    fd, an = np.array(fd), np.array(an)
    assert np.linalg.norm(fd - an) / np.linalg.norm(an) < 1e-4
    # latents: only touched ones have gradient; sample among them and a few untouched
    touched = np.flatnonzero(dl != 0)
    assert touched.size > 0
    idx = np.concatenate([rng.choice(touched, min(150, touched.size), replace=False),
                          rng.choice(np.flatnonzero(dl == 0), 10, replace=False)])
    fd, an = [], []
    for i in idx:
        lp, lm = lat.copy(), lat.copy()
        lp[i] = np.float32(lat[i] + 1e-5)
        lm[i] = np.float32(lat[i] - 1e-5)
        dlt = float(lp[i]) - float(lm[i])
        fd.append((L(lp, par) - L(lm, par)) / dlt)
        an.append(dl[i])
    fd, an = np.array(fd), np.array(an)
    assert np.linalg.norm(fd - an) / np.linalg.norm(an) < 1e-4
    assert np.all(an[-10:] == 0.0) and np.all(np.abs(fd[-10:]) < 1e-12)


def test_loss_is_mean_l2(O):
    """R17: loss = sum (y - R)^2 / (B c); with zero weights and output bias b3 the output
    is b3 everywhere, so the loss has the closed form mean((b3 - R)^2)."""
    d = Profile.named("ntc0.2", 32, 3)
    lat, par, chain = _material(O, d, 7)
    par[:] = 0.0
    b3 = np.array([0.25, 0.5, 0.75], np.float32)
    par[-3:] = b3
    ref = u8_to_f16_bits(chain[1])
    crops = gen_crops(1, 32, 1, 3, crop=8)
    loss, dp, dl = O.train_grads(d, lat, par, 1, crops, ref, 1, 1)
    R = ref.view(np.float16).astype(np.float64).reshape(16, 16, 3)
    vals = [R[y0:y0 + hh, x0:x0 + ww] for x0, y0, ww, hh in crops]
    want = np.mean(np.concatenate([((b3.astype(np.float16).astype(np.float64) - v) ** 2).reshape(-1, 3)
                                   for v in vals]))
    assert abs(loss - want) < 1e-15
    assert np.all(dl == 0.0)  # zero weights: no gradient reaches the latents


def test_channel_permutation_symmetry(O):
    """SPEC.md:296 / PAPER.md:377: permuting output channels (W3 rows, b3, reference
    channels) leaves the loss and the latent gradient unchanged."""
    d = Profile.named("ntc0.2", 32, 4)
    lat, par, chain = _material(O, d, 9)
    ref = u8_to_f16_bits(chain[0]).reshape(32, 32, 4)
    crops = gen_crops(2, 32, 0, 2, crop=16)
    perm = np.array([2, 0, 3, 1])
    P = O.num_params(d)
    W3o = P - (64 * 4 + 4)
    par2 = par.copy()
    par2[W3o:W3o + 256] = par[W3o:W3o + 256].reshape(4, 64)[perm].reshape(-1)
    par2[P - 4:] = par[P - 4:][perm]
    l1, _, dl1 = O.train_grads(d, lat, par, 0, crops, ref.reshape(-1), 3, 1)
    l2, _, dl2 = O.train_grads(d, lat, par2, 0, crops, np.ascontiguousarray(ref[..., perm]).reshape(-1), 3, 1)
    assert abs(l1 - l2) <= 1e-15 * max(1.0, abs(l1))
    assert np.allclose(dl1, dl2, rtol=1e-12, atol=1e-18)


def _centres(O, d, codes):
    """Bin centres of quantised codes, grid by grid: (code - (N/2 - 1)) Q."""
    cent = np.zeros(codes.shape, np.float32)
    for j in range(O.num_levels(d)):
        for k, B in ((0, d.b0), (1, d.b1)):
            a = O.grid_offset(d, j, k)
            b = O.grid_offset(d, j, 1) if k == 0 else O.grid_offset(d, j + 1, 0)
            cent[a:b] = (codes[a:b].astype(np.float64) - (2**B // 2 - 1)) / 2**B
    return cent


@pytest.mark.parametrize("mip", [0, 2, 4])
def test_noise_off_equals_quantised_path_on_centres(O, mip):
    """Pins train_grads' fp16-rounded forward (round_f16 = 1, the R14 path the GPU parity runs
    against) to the decode oracle: with latents at bin centres and noise off, the training
    forward reads exactly the decode's dequantised values (R25), so with the gain-0.3 weight
    recipe (no output clamps -- asserted) the loss equals mean((y - R)^2) of the decoded
    texels, and db3 equals its per-channel form 2/(B c) sum (y_k - R_k) (R17)."""
    d = Profile.named("ntc0.2", 32, 3)
    lat = gen_latents(21, O.num_latents(d))
    par = gen_weights_f32(22, d.input_dim, d.channels, 1, out_gain=0.3)
    chain = box_mip_chain_u8(gen_reference_u8(23, 32, 3))
    cent = _centres(O, d, O.quantize_latents(d, lat))
    codes = O.quantize_latents(d, cent)
    assert np.array_equal(_centres(O, d, codes), cent)   # centres are fixed points
    par16 = par.astype(np.float16)
    wm = 32 >> mip
    ref = u8_to_f16_bits(chain[mip])
    crops = np.array([[0, 0, wm, wm]], np.int32)
    loss, dp, dl = O.train_grads(d, cent, par16.astype(np.float32), mip, crops, ref, 0, 0, noise_on=False)
    q = np.stack(np.meshgrid(np.arange(wm), np.arange(wm), indexing="xy"), -1).reshape(-1, 2)
    q = np.concatenate([q, np.full((q.shape[0], 1), mip, np.int64)], 1).astype(np.int32)
    y = O.decode_texels(d, codes, par16.view(np.uint16), q)
    R = ref.view(np.float16).astype(np.float64).reshape(-1, 3)
    assert np.all((y > 0) & (y < 1))     # no clamp: decode == unclamped forward
    assert abs(loss - np.mean((y - R) ** 2)) < 1e-14
    assert np.allclose(dp[-3:], 2.0 / y.size * np.sum(y - R, 0), rtol=1e-10, atol=1e-15)


def test_quantize_latents_per_grid_bits(O):
    """ntco_quantize_latents assigns each grid its own B (G0: B0, G1: B1; Table 2): compared
    with the closed-form rule idx = clamp(floor(v 2^B + 1/2), -(N/2 - 1), N/2), code = idx +
    N/2 - 1 (R9/R10), evaluated in numpy on grid spans computed here from
    the grid resolutions (Table 1 geometry), for profiles whose B0 and B1 differ."""
    for name in ("ntc0.2", "ntc0.5", "ntc1.0", "ntc2.25"):
        d = Profile.named(name, 64, 4)
        lat = gen_latents(31, O.num_latents(d), scale=0.6)   # spans both clamp ends
        got = O.quantize_latents(d, lat)
        want = np.zeros_like(got)
        off = 0
        for j in range(O.num_levels(d)):
            r0, r1 = O.grid_res(d, j)
            for n, B in ((r0 * r0 * d.c0, d.b0), (r1 * r1 * d.c1, d.b1)):
                N = 2**B
                v = lat[off:off + n].astype(np.float64)
                idx = np.clip(np.floor(v * N + 0.5), -(N // 2 - 1), N // 2)
                want[off:off + n] = (idx + N // 2 - 1).astype(np.uint8)
                off += n
        assert off == lat.size
        assert np.array_equal(got, want), name


def test_adam_matches_torch(O):
    """Dense Adam vs torch.optim.Adam in fp64 over 5 steps (fp32 state)."""
    rng = np.random.default_rng(0)
    n = 1000
    p = rng.normal(0, 0.1, n).astype(np.float32)
    m = np.zeros(n, np.float32)
    v = np.zeros(n, np.float32)
    tp = torch.tensor(p.astype(np.float64), requires_grad=True)
    opt = torch.optim.Adam([tp], lr=0.005, betas=(0.9, 0.999), eps=1e-8)
    for t in range(1, 6):
        g = rng.normal(0, 1e-3, n).astype(np.float32)
        O.adam(p, m, v, g, t, 0.005)
        tp.grad = torch.tensor(g.astype(np.float64))
        opt.step()
        assert np.allclose(p, tp.detach().numpy(), atol=1e-6, rtol=1e-5)


def test_adam_first_step_closed_form_sparse_and_clamp(O):
    """t = 1 from zero state: p1 = p0 - lr g / (|g| + eps); sparse mode leaves g == 0
    entries untouched (R18); the clamp keeps latents in [lo, hi]."""
    rng = np.random.default_rng(1)
    n = 500
    p = rng.uniform(-0.3, 0.45, n).astype(np.float32)
    g = rng.normal(0, 1e-2, n).astype(np.float32)
    g[::3] = 0.0
    p0 = p.copy()
    m = np.zeros(n, np.float32)
    v = np.zeros(n, np.float32)
    lo, hi = O.quant_range(2)
    O.adam(p, m, v, g, 1, 0.1, sparse=True, clamp=(lo, hi))
    gd = g.astype(np.float64)
    want = np.clip(p0 - 0.1 * gd / (np.abs(gd) + 1e-8), lo, hi).astype(np.float32)
    nz = g != 0
    assert np.allclose(p[nz], want[nz], atol=1e-7)
    assert np.array_equal(p[~nz], p0[~nz]) and np.all(m[~nz] == 0) and np.all(v[~nz] == 0)
    assert p.min() >= lo and p.max() <= hi


def test_decode_mip_equals_decode_texels(O):
    """batch decode equals per-texel random-access decode exactly."""
    d = Profile.named("ntc0.2", 64, 8)
    grids = []
    for j in range(O.num_levels(d)):
        r0, r1 = O.grid_res(d, j)
        grids += [(r0 * r0 * d.c0, d.b0), (r1 * r1 * d.c1, d.b1)]
    codes = gen_codes(1, grids)
    w = gen_weights_f16(2, d.input_dim, 8)
    for m in (0, 2, 5):
        img = O.decode_mip(d, codes, w, m)
        wm = 64 >> m
        q = np.array([[x, y, m] for y in range(wm) for x in range(wm)], np.int32)
        assert np.array_equal(O.decode_texels(d, codes, w, q).reshape(img.shape), img)


def test_decode_composition_from_library_routines(O):
    """Independent decode from library routines: torch grid_sample (G1 bilinear) and
    nearest-cell gathers (G0) on dequantised grids, the triangle-wave Fourier series (PE),
    numpy float16 (LOD, input rounding), torch Linear + hardswish(2x)/2 (MLP), clamp."""
    d = Profile.named("ntc0.2", 32, 8)
    L = O.num_levels(d)
    grids = []
    for j in range(L):
        r0, r1 = O.grid_res(d, j)
        grids += [(r0 * r0 * d.c0, d.b0), (r1 * r1 * d.c1, d.b1)]
    codes = gen_codes(5, grids)
    wf = gen_weights_f16(6, d.input_dim, 8, out_gain=1.0)
    w = wf.view(np.float16).astype(np.float64)
    M = O.num_mips(32)
    ks = np.arange(1, 20001, 2, dtype=np.float64)

    def tri(t):
        return 8 / math.pi**2 * np.sum(np.cos(2 * math.pi * ks * t) / ks**2)

    def deq(c, B):
        return (c.astype(np.float64) - (2**B // 2 - 1)) / 2**B

    for m in range(M):
        wm = 32 >> m
        j = O.level_of_mip(d, m)
        r0, r1 = O.grid_res(d, j)
        g0 = deq(codes[O.grid_offset(d, j, 0):][: r0 * r0 * 8].reshape(r0, r0, 8), 2)
        g1 = deq(codes[O.grid_offset(d, j, 1):][: r1 * r1 * 12].reshape(r1, r1, 12), 4)
        ys, xs = np.meshgrid(np.arange(wm), np.arange(wm), indexing="ij")
        grid = torch.tensor(np.stack([(xs + 0.5) / wm * 2 - 1, (ys + 0.5) / wm * 2 - 1], -1)[None])
        s1 = torch.nn.functional.grid_sample(torch.tensor(g1.transpose(2, 0, 1)[None]), grid, mode="bilinear",
                                             padding_mode="border", align_corners=False)[0].numpy()
        X = np.zeros((wm, wm, d.input_dim))
        for y in range(wm):
            for x in range(wm):
                # G0 taps: the cells whose centres bracket the texel centre (clamped)
                cx = (x + 0.5) * r0 / wm - 0.5
                cy = (y + 0.5) * r0 / wm - 0.5
                ix, iy = math.floor(cx), math.floor(cy)
                taps = [(ix, iy), (ix + 1, iy), (ix, iy + 1), (ix + 1, iy + 1)]
                feats = [g0[min(max(b, 0), r0 - 1), min(max(a, 0), r0 - 1)] for a, b in taps]
                pe = []
                for p in (x % 8, y % 8):
                    for h in range(3):
                        pe += [tri(2**h * p / 8), tri(2**h * p / 8 - 0.25)]
                X[y, x] = np.concatenate(feats + [s1[:, y, x], np.rint(2 * np.array(pe)) / 2, [m / (M - 1)]])
        X = X.astype(np.float16).astype(np.float64).reshape(-1, d.input_dim)
        dims = [(d.input_dim, 64), (64, 64), (64, 8)]
        off, h = 0, torch.tensor(X)
        for li, (fi, fo) in enumerate(dims):
            W = torch.tensor(w[off: off + fi * fo].reshape(fo, fi)); off += fi * fo
            b = torch.tensor(w[off: off + fo]); off += fo
            h = torch.nn.functional.linear(h, W, b)
            if li < 2:
                h = torch.nn.functional.hardswish(2 * h) / 2
        want = h.clamp(0, 1).numpy().reshape(wm, wm, 8)
        got = O.decode_mip(d, codes, wf, m)
        assert np.allclose(got, want, atol=1e-12, rtol=0), m
