"""GPU parity of the training step (t1..t8) against the CPU oracle, through the C ABI.

Bar (BASELINE.json north_star): relative error <= 1e-2 on gradients (per tensor, R21:
||g - g_ref|| / ||g_ref|| <= 1e-2 and max |g - g_ref| <= 1e-2 max |g_ref|); the noise
values are bit-exact; the optimizer step matches the oracle's Adam on identical gradients.
"""
import numpy as np
import pytest
import torch

import paper_2305_17105_b200 as ntc
from paper_2305_17105_b200.synth import (Profile, box_mip_chain_u8, gen_crops, gen_grads, gen_latents,
                                         gen_reference_u8, gen_weights_f32, u8_to_f16_bits)

pytestmark = pytest.mark.gpu
DEV = "cuda:0"
REL = 1e-2


def _setup(O, W, c, seed, mip, n_crops, crop, out_gain=1.0, activation=0, hidden_mats=1, profile="ntc0.2"):
    d = Profile.named(profile, W, c, hidden_mats, activation)
    lat = gen_latents(seed, O.num_latents(d))
    par = gen_weights_f32(seed + 1, d.input_dim, c, hidden_mats, out_gain=out_gain)
    chain = box_mip_chain_u8(gen_reference_u8(seed + 2, W, c))
    ref = u8_to_f16_bits(chain[mip])
    crops = gen_crops(seed + 3, W, mip, n_crops, crop)
    return d, lat, par, ref, crops


def _gpu_buffers(O, d, lat, par):
    NL, P = O.num_latents(d), O.num_params(d)
    t = {k: torch.zeros(NL, device=DEV) for k in ("m_lat", "v_lat", "grad_lat", "noisy")}
    t.update({k: torch.zeros(P, device=DEV) for k in ("m_par", "v_par", "grad_par")})
    t["latents"] = torch.from_numpy(lat.copy()).to(DEV)
    t["params"] = torch.from_numpy(par.copy()).to(DEV)
    return t


def _gpu_grads(O, d, lat, par, ref, crops, mip, seed, step, noise_on=True):
    tr = ntc.Trainer(d)
    t = _gpu_buffers(O, d, lat, par)
    refd = torch.from_numpy(ref.view(np.int16)).to(DEV)
    batch = ntc.make_batch(mip, crops, refd, (d.width >> mip) * d.channels)
    hp = ntc.Hparams(0.01, 0.005, 0.9, 0.999, 1e-8, step, seed, int(noise_on), 0)
    loss = torch.zeros(1, device=DEV)
    st = torch.zeros(1, dtype=torch.int32, device=DEV)
    ntc.ntc_train_step(tr, ntc.make_buffers(t), batch, hp, loss, st, flags=ntc.NTC_STEP_GRADS)
    torch.cuda.synchronize()
    assert st.item() == 0
    return loss.item(), t["grad_par"].cpu().numpy().astype(np.float64), t["grad_lat"].cpu().numpy().astype(
        np.float64), t


def _param_slices(d):
    D, c = d.input_dim, d.channels
    names, sizes = ["W1", "b1", "W2", "b2"], [64 * D, 64, 4096, 64]
    if d.hidden_mats == 2:
        names, sizes = names + ["W2b", "b2b"], sizes + [4096, 64]
    names, sizes = names + ["W3", "b3"], sizes + [64 * c, c]
    out, o = {}, 0
    for n, s in zip(names, sizes):
        out[n] = slice(o, o + s)
        o += s
    return out


def _check_grad(name, g, ref):
    nref = np.linalg.norm(ref)
    assert nref > 0, name
    rel = np.linalg.norm(g - ref) / nref
    mx = np.abs(g - ref).max() / np.abs(ref).max()
    assert rel <= REL and mx <= REL, (name, rel, mx)
    return rel


def _check_all(O, d, gp, gl, dp, dl):
    for n, sl in _param_slices(d).items():
        _check_grad(n, gp[sl], dp[sl])
    for j in range(O.num_levels(d)):
        for k in range(2):
            a = O.grid_offset(d, j, k)
            b = O.grid_offset(d, j, 1) if k == 0 else O.grid_offset(d, j + 1, 0)
            if np.any(dl[a:b] != 0):
                _check_grad(f"G{j}.{k}", gl[a:b], dl[a:b])
            else:
                assert np.all(gl[a:b] == 0)


@pytest.mark.parametrize("mip,n_crops,crop", [(0, 2, 32), (1, 3, 16), (2, 4, 8), (4, 1, 4), (5, 2, 2), (0, 3, 24), (1, 2, 20)])
def test_train_grads_small(O, mip, n_crops, crop):
    """Loss and every gradient tensor vs the oracle on a 64^2 x 8 material, at several LODs
    (crops smaller than a tile, ragged last tiles, overlapping crops)."""
    d, lat, par, ref, crops = _setup(O, 64, 8, 10 + mip, mip, n_crops, crop)
    loss, gp, gl, _ = _gpu_grads(O, d, lat, par, ref, crops, mip, 77, 5)
    loss_o, dp, dl = O.train_grads(d, lat, par, mip, crops, ref, 77, 5)
    assert abs(loss - loss_o) <= 1e-3 * loss_o
    _check_all(O, d, gp, gl, dp, dl)


@pytest.mark.parametrize("mip,n_crops,crop", [(0, 2, 32), (3, 2, 8)])
def test_train_grads_gelu(O, mip, n_crops, crop):
    """f4: the exact-GELU variant (activation = 1) of the training step: loss
    and every gradient tensor vs the oracle."""
    d, lat, par, ref, crops = _setup(O, 64, 9, 40 + mip, mip, n_crops, crop, activation=1)
    loss, gp, gl, _ = _gpu_grads(O, d, lat, par, ref, crops, mip, 41, 2)
    loss_o, dp, dl = O.train_grads(d, lat, par, mip, crops, ref, 41, 2)
    assert abs(loss - loss_o) <= 1e-3 * loss_o
    _check_all(O, d, gp, gl, dp, dl)


@pytest.mark.parametrize("mip,n_crops,crop,act", [(0, 2, 32, 0), (2, 3, 8, 0), (0, 2, 24, 1)])
def test_train_grads_depth2(O, mip, n_crops, crop, act):
    """f4: depth reading B ([D,64,64,64,c], hidden_mats = 2, R11) of the training step (one
    slot per CTA): loss and every gradient tensor, including W2b/b2b, vs the oracle."""
    d, lat, par, ref, crops = _setup(O, 64, 9, 60 + mip, mip, n_crops, crop, activation=act, hidden_mats=2)
    loss, gp, gl, _ = _gpu_grads(O, d, lat, par, ref, crops, mip, 61, 3)
    loss_o, dp, dl = O.train_grads(d, lat, par, mip, crops, ref, 61, 3)
    assert abs(loss - loss_o) <= 1e-3 * loss_o
    _check_all(O, d, gp, gl, dp, dl)


@pytest.mark.parametrize("profile,mip,hm,act", [("ntc0.5", 0, 1, 0), ("ntc0.5", 2, 1, 0), ("ntc1.0", 0, 1, 0),
                                                ("ntc1.0", 3, 1, 1), ("ntc2.25", 0, 1, 0), ("ntc2.25", 1, 2, 0)])
def test_train_grads_other_profiles(O, profile, mip, hm, act):
    """f4: the K1 = 80/96 profiles of Table 2 (X in two K atoms, one slot per CTA): loss and
    every gradient tensor vs the oracle, at several LODs, depths and activations."""
    d, lat, par, ref, crops = _setup(O, 64, 9, 80 + mip, mip, 2, 24 >> min(mip, 2), activation=act, hidden_mats=hm,
                                     profile=profile)
    loss, gp, gl, _ = _gpu_grads(O, d, lat, par, ref, crops, mip, 81, 2)
    loss_o, dp, dl = O.train_grads(d, lat, par, mip, crops, ref, 81, 2)
    assert abs(loss - loss_o) <= 1e-3 * loss_o
    _check_all(O, d, gp, gl, dp, dl)


def test_train_grads_c9_256(O):
    d, lat, par, ref, crops = _setup(O, 256, 9, 3, 0, 4, 64)
    loss, gp, gl, _ = _gpu_grads(O, d, lat, par, ref, crops, 0, 5, 1)
    loss_o, dp, dl = O.train_grads(d, lat, par, 0, crops, ref, 5, 1)
    assert abs(loss - loss_o) <= 1e-3 * loss_o
    _check_all(O, d, gp, gl, dp, dl)


def test_train_grads_full_size_c4(O):
    """configs[3] at full size in the bench launch configuration: 4096^2 x 9, 4 random 256^2
    crops at LOD 0 (262,144 texels), one GRADS call vs the oracle's full-batch gradients."""
    d, lat, par, ref, crops = _setup(O, 4096, 9, 0x4E544303, 0, 4, 256, out_gain=0.3)
    loss, gp, gl, _ = _gpu_grads(O, d, lat, par, ref, crops, 0, 0x4E544303, 1)
    loss_o, dp, dl = O.train_grads(d, lat, par, 0, crops, ref, 0x4E544303, 1)
    assert abs(loss - loss_o) <= 1e-3 * loss_o
    _check_all(O, d, gp, gl, dp, dl)


def test_noise_bit_exact(O):
    """t2: noisy latents = fp16(fp32(latent + U(-Q/2,Q/2))) with the oracle's Philox draws,
    bit-exact, written exactly over the footprint (the buffer holds fp16, R14)."""
    d, lat, par, ref, crops = _setup(O, 64, 8, 4, 0, 2, 16)
    _, _, _, t = _gpu_grads(O, d, lat, par, ref, crops, 0, 1234, 9)
    noisy = t["noisy"].cpu().view(torch.float16).numpy()[: lat.size]
    touched = np.flatnonzero(noisy != 0)
    assert touched.size > 0
    for i in touched[:: max(1, touched.size // 500)]:
        B = d.b0 if any(O.grid_offset(d, j, 0) <= i < O.grid_offset(d, j, 1) for j in range(O.num_levels(d))) \
            else d.b1
        want = np.float16(np.float32(lat[i]) + np.float32(O.noise(1234, 9, int(i), B)))
        assert noisy[i] == want


def test_adam_apply_parity(O):
    """t8 in isolation: identical synthetic gradients (zeros included) -> Adam on the weights
    (dense) and on the footprint latents (sparse, g == 0 skipped) + clamp, vs the oracle."""
    d, lat, par, ref, crops = _setup(O, 64, 8, 6, 0, 2, 16)
    NL, P = O.num_latents(d), O.num_params(d)
    # oracle footprint: latents read by the crops' texels
    fp = np.zeros(NL, bool)
    for x0, y0, w, h in crops:
        for y in range(y0, y0 + h):
            for x in range(x0, x0 + w):
                ti, _ = O.address(d, 0, x, y)
                r0, r1 = O.grid_res(d, ti[0])
                for t in range(4):
                    a = O.grid_offset(d, ti[0], 0) + (ti[2 + 2 * t] * r0 + ti[1 + 2 * t]) * d.c0
                    fp[a: a + d.c0] = True
                    b = O.grid_offset(d, ti[0], 1) + (ti[10 + 2 * t] * r1 + ti[9 + 2 * t]) * d.c1
                    fp[b: b + d.c1] = True
    gl = gen_grads(8, NL, 1e-3)
    gl[~fp] = 0.0
    gp = gen_grads(9, P, 1e-2, zero_frac=0.0)
    t = _gpu_buffers(O, d, lat, par)
    m0 = gen_grads(10, NL, 1e-4, 0.0)
    v0 = np.abs(gen_grads(11, NL, 1e-6, 0.0))
    t["grad_lat"].copy_(torch.from_numpy(gl))
    t["grad_par"].copy_(torch.from_numpy(gp))
    t["m_lat"].copy_(torch.from_numpy(m0))
    t["v_lat"].copy_(torch.from_numpy(v0))
    tr = ntc.Trainer(d)
    refd = torch.from_numpy(ref.view(np.int16)).to(DEV)
    batch = ntc.make_batch(0, crops, refd, 64 * 8)
    hp = ntc.Hparams(0.01, 0.005, 0.9, 0.999, 1e-8, 3, 1, 1, 0)
    ntc.ntc_train_step(tr, ntc.make_buffers(t), batch, hp, torch.zeros(1, device=DEV), flags=ntc.NTC_STEP_APPLY)
    torch.cuda.synchronize()
    # oracle
    p_o, m_o, v_o = par.copy(), np.zeros(P, np.float32), np.zeros(P, np.float32)
    O.adam(p_o, m_o, v_o, gp, 3, 0.005)
    assert np.allclose(t["params"].cpu().numpy(), p_o, rtol=1e-5, atol=1e-6)
    lo = {}
    for j in range(O.num_levels(d)):
        for k, B in ((0, d.b0), (1, d.b1)):
            a = O.grid_offset(d, j, k)
            b = O.grid_offset(d, j, 1) if k == 0 else O.grid_offset(d, j + 1, 0)
            l_o, mm, vv = lat[a:b].copy(), m0[a:b].copy(), v0[a:b].copy()
            O.adam(l_o, mm, vv, gl[a:b].copy(), 3, 0.01, sparse=True, clamp=O.quant_range(B))
            assert np.allclose(t["latents"].cpu().numpy()[a:b], l_o, rtol=1e-5, atol=1e-6), (j, k)
            assert np.allclose(t["m_lat"].cpu().numpy()[a:b], mm, rtol=1e-5, atol=1e-9)
            assert np.allclose(t["v_lat"].cpu().numpy()[a:b], vv, rtol=1e-5, atol=1e-12)


def test_train_loop_tracks_oracle(O):
    """Three full GRADS+APPLY steps: the loss trajectory follows the oracle's (oracle
    gradients -> fp32 -> oracle Adam), and all latents stay inside their quantisation range."""
    d, lat, par, ref, crops0 = _setup(O, 64, 8, 21, 0, 2, 32)
    tr = ntc.Trainer(d)
    t = _gpu_buffers(O, d, lat, par)
    refd = torch.from_numpy(ref.view(np.int16)).to(DEV)
    NL, P = O.num_latents(d), O.num_params(d)
    lat_o, par_o = lat.copy(), par.copy()
    st_o = [np.zeros(NL, np.float32), np.zeros(NL, np.float32), np.zeros(P, np.float32), np.zeros(P, np.float32)]
    for step in range(1, 4):
        crops = gen_crops(100 + step, 64, 0, 2, 32)
        batch = ntc.make_batch(0, crops, refd, 64 * 8)
        hp = ntc.Hparams(0.01, 0.005, 0.9, 0.999, 1e-8, step, 3, 1, 0)
        loss = torch.zeros(1, device=DEV)
        ntc.ntc_train_step(tr, ntc.make_buffers(t), batch, hp, loss)
        torch.cuda.synchronize()
        lo, dp, dl = O.train_grads(d, lat_o, par_o, 0, crops, ref, 3, step)
        assert abs(loss.item() - lo) <= 2e-2 * lo, (step, loss.item(), lo)
        O.adam(par_o, st_o[2], st_o[3], dp.astype(np.float32), step, 0.005)
        for j in range(O.num_levels(d)):
            for k, B in ((0, d.b0), (1, d.b1)):
                a = O.grid_offset(d, j, k)
                b = O.grid_offset(d, j, 1) if k == 0 else O.grid_offset(d, j + 1, 0)
                sl = slice(a, b)
                lv, mv, vv = lat_o[sl].copy(), st_o[0][sl].copy(), st_o[1][sl].copy()
                O.adam(lv, mv, vv, dl[sl].astype(np.float32), step, 0.01, sparse=True, clamp=O.quant_range(B))
                lat_o[sl], st_o[0][sl], st_o[1][sl] = lv, mv, vv
                g = t["latents"].cpu().numpy()[sl]
                lo_b, hi_b = O.quant_range(B)
                assert g.min() >= lo_b and g.max() <= hi_b


def test_nonfinite_loss_sets_status(O):
    d, lat, par, ref, crops = _setup(O, 64, 8, 1, 0, 1, 16)
    par = par.copy()
    par[-8:] = np.inf
    tr = ntc.Trainer(d)
    t = _gpu_buffers(O, d, lat, par)
    refd = torch.from_numpy(ref.view(np.int16)).to(DEV)
    st = torch.zeros(1, dtype=torch.int32, device=DEV)
    ntc.ntc_train_step(tr, ntc.make_buffers(t), ntc.make_batch(0, crops, refd, 512),
                       ntc.Hparams(0.01, 0.005, 0.9, 0.999, 1e-8, 1, 1, 1, 0), torch.zeros(1, device=DEV), st,
                       flags=ntc.NTC_STEP_GRADS)
    torch.cuda.synchronize()
    assert st.item() & ntc.NTC_ERR_NONFINITE


def test_fused_grads_apply_equals_split_calls(O):
    """GRADS|APPLY in one call (reduction and Adam share a launch) equals a GRADS call followed
    by an APPLY call: bit-identical weights and weight moments (the weight-gradient reduction
    is deterministic); the latents to fp32 rounding (the latent-gradient scatter uses float
    atomics, whose summation order varies between runs)."""
    d, lat, par, ref, crops = _setup(O, 128, 9, 77, 0, 3, 40)
    refd = torch.from_numpy(ref.view(np.int16)).to(DEV)
    out = []
    for split in (False, True):
        tr = ntc.Trainer(d)
        t = _gpu_buffers(O, d, lat, par)
        bufs = ntc.make_buffers(t)
        for step in (1, 2):
            hp = ntc.Hparams(0.01, 0.005, 0.9, 0.999, 1e-8, step, 5, 1, 0)
            batch = ntc.make_batch(0, gen_crops(300 + step, 128, 0, 3, 40), refd, 128 * 9)
            loss = torch.zeros(1, device=DEV)
            if split:
                ntc.ntc_train_step(tr, bufs, batch, hp, loss, flags=ntc.NTC_STEP_GRADS)
                ntc.ntc_train_step(tr, bufs, batch, hp, loss, flags=ntc.NTC_STEP_APPLY)
            else:
                ntc.ntc_train_step(tr, bufs, batch, hp, loss)
        torch.cuda.synchronize()
        out.append({k: t[k].cpu().numpy().copy() for k in ("params", "m_par", "v_par", "latents", "m_lat", "v_lat")})
    for k in ("params", "m_par", "v_par"):
        assert np.array_equal(out[0][k], out[1][k]), k
    for k in ("latents", "m_lat", "v_lat"):
        assert np.allclose(out[0][k], out[1][k], rtol=1e-4, atol=1e-9), k


def test_train_step_cuda_graph_capture(O):
    """A training step is CUDA-graph capturable: no host synchronisation or allocation on the
    hot path (the bench / DP step can be replayed as a graph).  A graph of two steps (GRADS|APPLY,
    then the split GRADS + APPLY calls of the data-parallel mode) replayed twice equals the same
    four calls made directly, to fp32 rounding: the latent-gradient scatter's float atomics
    make the latents run-order dependent in their last bits, and through the fp16 rounding of
    the next step's inputs the weight updates too."""
    d, lat, par, ref, crops = _setup(O, 128, 9, 78, 0, 3, 40)
    refd = torch.from_numpy(ref.view(np.int16)).to(DEV)
    batch = ntc.make_batch(0, gen_crops(400, 128, 0, 3, 40), refd, 128 * 9)
    hp = ntc.Hparams(0.01, 0.005, 0.9, 0.999, 1e-8, 3, 5, 1, 0)
    out = []
    for graph in (False, True):
        tr = ntc.Trainer(d)
        t = _gpu_buffers(O, d, lat, par)
        bufs = ntc.make_buffers(t)
        loss = torch.zeros(1, device=DEV)

        def two_steps():
            ntc.ntc_train_step(tr, bufs, batch, hp, loss)
            ntc.ntc_train_step(tr, bufs, batch, hp, loss, flags=ntc.NTC_STEP_GRADS)
            ntc.ntc_train_step(tr, bufs, batch, hp, loss, flags=ntc.NTC_STEP_APPLY)

        if graph:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                two_steps()
            for _ in range(2):
                g.replay()
        else:
            for _ in range(2):
                two_steps()
        torch.cuda.synchronize()
        out.append({k: t[k].cpu().numpy().copy() for k in ("params", "m_par", "latents")})
    for k in ("params", "m_par"):
        assert np.allclose(out[0][k], out[1][k], rtol=1e-5, atol=1e-8), k
    assert np.allclose(out[0]["latents"], out[1]["latents"], rtol=1e-4, atol=1e-9)
