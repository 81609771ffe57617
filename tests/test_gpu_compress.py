"""GPU run of the compression loop (f1): training lowers the loss, the frozen phase leaves
the latents exactly at their bin centres, and decoding the compressed material reproduces
the training forward (same quantised latents, same fp16 weights)."""
import numpy as np
import pytest
import torch

import paper_2305_17105_b200 as ntc
from paper_2305_17105_b200.compress import CompressConfig, Compressor
from paper_2305_17105_b200.synth import Profile, box_mip_chain_u8, gen_reference_u8, u8_to_f16_bits

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def test_compress_small_material(O):
    d = Profile.named("ntc0.2", 64, 4)
    chain = [torch.from_numpy(u8_to_f16_bits(m).view(np.int16).copy()).to(DEV)
             for m in box_mip_chain_u8(gen_reference_u8(5, 64, 4))]
    cfg = CompressConfig(steps=1500, crops=4, crop=32, seed=11)
    comp = Compressor(d, chain, cfg, DEV)
    codes, w16 = comp.run(log_every=50)
    losses = [l for _, l in comp.losses]
    assert np.mean(losses[-5:]) < 0.5 * np.mean(losses[:3]), losses[:3] + losses[-5:]
    # frozen latents are bin centres
    lat = comp.t["latents"].cpu().numpy()
    cod = codes.cpu().numpy()
    for j in range(O.num_levels(d)):
        for k, B in ((0, d.b0), (1, d.b1)):
            a = O.grid_offset(d, j, k)
            b = O.grid_offset(d, j, 1) if k == 0 else O.grid_offset(d, j + 1, 0)
            assert np.array_equal(lat[a:b], ((cod[a:b].astype(np.int64) - (2**B // 2 - 1)) / 2**B).astype(np.float32))
    # decode the compressed material; compare with a frozen, noise-free training forward
    mat = ntc.Material(d, codes, w16.view(torch.int16))
    out = torch.empty((64, 64, 4), dtype=torch.float16, device=DEV)
    ntc.ntc_decode_mip(mat, 0, out)
    ref = chain[0].view(torch.float16).float().view(64, 64, 4)
    mse_decode = torch.mean((out.float() - ref) ** 2).item()
    batch = ntc.make_batch(0, np.array([[0, 0, 64, 64]], np.int32), chain[0], 64 * 4)
    hp = ntc.Hparams(0.0, 0.0, 0.9, 0.999, 1e-8, 1, 0, 0, 0, 1)
    loss = torch.zeros(1, device=DEV)
    ntc.ntc_train_step(comp.trainer, comp.buf, batch, hp, loss, flags=ntc.NTC_STEP_GRADS)
    torch.cuda.synchronize()
    assert abs(loss.item() - mse_decode) <= 0.05 * mse_decode + 2e-6, (loss.item(), mse_decode)
    psnr = -10 * np.log10(mse_decode)
    assert psnr > 20.0


def _state(t):
    return {k: t[k].cpu().numpy().copy() for k in ("latents", "params", "m_lat", "v_lat", "m_par", "v_par")}


def _check_weight_grads(d, gp, dp):
    from test_gpu_train import _check_grad, _param_slices

    for n, sl in _param_slices(d).items():
        _check_grad(n, gp[sl], dp[sl])


def _oracle_apply(O, d, s, gp, gl, fp, hp, frozen):
    """The oracle's t8 from state `s` on the GPU's own gradients (Adam parity is a separate
    pin; this isolates the loop's schedule): dense Adam on the weights; footprint-sparse Adam
    + clamp on the latents, or nothing when frozen (R25)."""
    from helpers import grid_spans

    p, m, v = s["params"].copy(), s["m_par"].copy(), s["v_par"].copy()
    O.adam(p, m, v, gp.astype(np.float32), hp.step, hp.lr_weight)
    lat, ml, vl = s["latents"].copy(), s["m_lat"].copy(), s["v_lat"].copy()
    if not frozen:
        g = np.where(fp, gl, 0.0).astype(np.float32)
        for sl, B in grid_spans(O, d):
            a, b, c = lat[sl].copy(), ml[sl].copy(), vl[sl].copy()
            O.adam(a, b, c, g[sl].copy(), hp.step, hp.lr_latent, sparse=True, clamp=O.quant_range(B))
            lat[sl], ml[sl], vl[sl] = a, b, c
    return p, m, v, lat, ml, vl


def test_frozen_phase_vs_oracle(O):
    """f1 frozen phase (R25): latents at bin centres, noise off, latents frozen.
    The GRADS call's weight gradients match the oracle's noise-free gradients (rel 1e-2 per
    tensor, R21), no latent gradient is scattered, and APPLY leaves latents and their Adam
    moments bit-identical while the weights take the oracle's Adam step."""
    from helpers import centres, oracle_footprint

    from test_gpu_train import _gpu_buffers, _setup

    for mip, n_crops, crop in ((0, 2, 32), (2, 3, 8)):
        d, lat, par, ref, crops = _setup(O, 64, 8, 90 + mip, mip, n_crops, crop, out_gain=0.3)
        cent = centres(O, d, O.quantize_latents(d, lat))
        t = _gpu_buffers(O, d, cent, par)
        t["m_lat"].fill_(1e-4)   # nonzero moments: APPLY must not touch them either
        t["v_lat"].fill_(1e-8)
        s0 = _state(t)
        tr = ntc.Trainer(d)
        refd = torch.from_numpy(ref.view(np.int16)).to(DEV)
        batch = ntc.make_batch(mip, crops, refd, (64 >> mip) * 8)
        hp = ntc.Hparams(0.01, 0.005, 0.9, 0.999, 1e-8, 4, 17, 0, 0, 1)
        loss = torch.zeros(1, device=DEV)
        bufs = ntc.make_buffers(t)
        ntc.ntc_train_step(tr, bufs, batch, hp, loss, flags=ntc.NTC_STEP_GRADS)
        torch.cuda.synchronize()
        loss_o, dp, dl = O.train_grads(d, cent, par, mip, crops, ref, 17, 4, noise_on=False)
        assert abs(loss.item() - loss_o) <= 1e-3 * loss_o
        gp = t["grad_par"].cpu().numpy().astype(np.float64)
        _check_weight_grads(d, gp, dp)
        assert np.all(t["grad_lat"].cpu().numpy() == 0.0)
        ntc.ntc_train_step(tr, bufs, batch, hp, loss, flags=ntc.NTC_STEP_APPLY)
        torch.cuda.synchronize()
        s1 = _state(t)
        for k in ("latents", "m_lat", "v_lat"):
            assert np.array_equal(s1[k], s0[k]), k
        p, m, v, *_ = _oracle_apply(O, d, s0, gp, None, oracle_footprint(O, d, mip, crops), hp, True)
        assert np.allclose(s1["params"], p, rtol=1e-5, atol=1e-6)
        assert np.allclose(s1["m_par"], m, rtol=1e-5, atol=1e-9)


def test_compress_loop_vs_oracle_driven_loop(O):
    """f1 schedule step by step against an oracle-driven loop: every
    step's batch (LOD law, crops) and hyper-parameters (cosine LRs, noise, freeze) come from
    the Compressor's host schedule; from the same state, the oracle computes that step's loss
    and gradients (noisy phase: with the same Philox noise; frozen phase: noise off) and its
    Adam step, and the GPU's next state must match it.  At the switch the explicit
    quantisation must give the oracle's codes bit-exactly and put the latents at the oracle's
    bin centres."""
    from helpers import centres, oracle_footprint

    from test_gpu_train import _check_all

    d = Profile.named("ntc0.2", 32, 4)
    chain_u8 = box_mip_chain_u8(gen_reference_u8(12, 32, 4))
    ref16 = [u8_to_f16_bits(m) for m in chain_u8]
    chain = [torch.from_numpy(r.view(np.int16).copy()).to(DEV) for r in ref16]
    cfg = CompressConfig(steps=6, finetune_fraction=0.5, crops=2, crop=16, seed=13, uniform_lod_fraction=0.5)
    comp = Compressor(d, chain, cfg, DEV)
    assert comp.total == 9
    mips = []
    for i in range(comp.total):
        frozen = i >= cfg.steps
        if i == cfg.steps:
            lat_before = comp.t["latents"].cpu().numpy().copy()
            comp.freeze()
            codes = comp.codes.cpu().numpy()
            assert np.array_equal(codes, O.quantize_latents(d, lat_before))
            assert np.array_equal(comp.t["latents"].cpu().numpy(), centres(O, d, codes))
        s0 = _state(comp.t)
        batch, hp = comp.plan(frozen)
        mip, crops = batch[0].mip, batch[1].copy()
        mips.append(mip)
        assert hp.noise_on == (0 if frozen else 1) and hp.freeze_latents == (1 if frozen else 0)
        ntc.ntc_train_step(comp.trainer, comp.buf, batch, hp, comp.loss, flags=ntc.NTC_STEP_GRADS)
        torch.cuda.synchronize()
        loss_o, dp, dl = O.train_grads(d, s0["latents"], s0["params"], mip, crops, ref16[mip], cfg.seed, hp.step,
                                       noise_on=not frozen)
        assert abs(comp.loss.item() - loss_o) <= 1e-3 * loss_o, (i, comp.loss.item(), loss_o)
        gp = comp.t["grad_par"].cpu().numpy().astype(np.float64)
        gl = comp.t["grad_lat"].cpu().numpy().astype(np.float64)
        fp = oracle_footprint(O, d, mip, crops)
        if frozen:
            _check_weight_grads(d, gp, dp)
            assert np.all(gl[fp] == 0.0)
        else:
            _check_all(O, d, gp, np.where(fp, gl, 0.0), dp, dl)
        ntc.ntc_train_step(comp.trainer, comp.buf, batch, hp, comp.loss, flags=ntc.NTC_STEP_APPLY)
        torch.cuda.synchronize()
        s1 = _state(comp.t)
        p, m, v, lat, ml, vl = _oracle_apply(O, d, s0, gp, gl, fp, hp, frozen)
        assert np.allclose(s1["params"], p, rtol=1e-5, atol=1e-6), i
        assert np.allclose(s1["latents"], lat, rtol=1e-5, atol=1e-6), i
        assert np.allclose(s1["m_lat"], ml, rtol=1e-5, atol=1e-9), i
        if frozen:
            assert np.array_equal(s1["latents"], s0["latents"])
    assert len(set(mips)) > 1   # the LOD law drew more than one level
