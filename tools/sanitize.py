"""Small invocations of every product kernel, for compute-sanitizer (profiling/QA helper, not
product code).  Run ON the GPU box under each tool, e.g.

    compute-sanitizer --tool memcheck  python tools/sanitize.py
    compute-sanitizer --tool synccheck python tools/sanitize.py
    compute-sanitizer --tool racecheck python tools/sanitize.py --small
    compute-sanitizer --tool initcheck python tools/sanitize.py --small

Covers: material create (quantise / pack / weight image), C1 (256^2 c=8 mip 0) and C2 (2048^2
c=9 full chain) decodes, random queries with bad rows, multi-material decode, filtering, and a
training step (GRADS|APPLY, then the split GRADS / APPLY calls) with the depth-2 variant.
--small drops C2 to a 512^2 chain (racecheck / initcheck are slower)."""
from __future__ import annotations

import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2305_17105_b200 as ntc  # noqa: E402
from paper_2305_17105_b200.synth import (Profile, box_mip_chain_u8, gen_codes, gen_crops, gen_latents,  # noqa: E402
                                         gen_queries, gen_reference_u8, gen_weights_f16, gen_weights_f32,
                                         u8_to_f16_bits)

DEV = "cuda:0"


def material(d, seed):
    grids = []
    for j in range(ntc.ntc_num_levels(d)):
        r0, r1, _, _ = ntc.ntc_grid_layout(d, j)
        grids += [(r0 * r0 * d.c0, d.b0), (r1 * r1 * d.c1, d.b1)]
    codes = gen_codes(seed, grids)
    w = gen_weights_f16(seed + 1, d.input_dim, d.channels, d.hidden_mats)
    return ntc.Material(d, torch.from_numpy(codes).to(DEV), torch.from_numpy(w.view(np.int16)).to(DEV))


def decode_runs(small):
    # C1: 256^2, c = 8, mip 0
    d = Profile.named("ntc0.2", 256, 8)
    m = material(d, 1)
    out = torch.empty(256 * 256 * 8, dtype=torch.float16, device=DEV)
    ntc.ntc_decode_mip(m, 0, out)
    # C2: full chain (2048^2, c = 9; 512^2 with --small)
    W = 512 if small else 2048
    d2 = Profile.named("ntc0.2", W, 9)
    m2 = material(d2, 2)
    out2 = torch.empty(ntc.ntc_chain_texels(d2) * 9, dtype=torch.float16, device=DEV)
    ntc.ntc_decode_chain(m2, out2)
    # random queries incl. out-of-range rows (device status word)
    xym = torch.from_numpy(gen_queries(3, W, 4099).astype(np.int64))
    xym[7, 0] = W + 3  # x out of range at mip 0 (device status word, NaN row)
    xym[7, 2] = 0
    q = ntc.pack_queries(xym).to(DEV)
    qo = torch.empty(q.numel() * 9, dtype=torch.float16, device=DEV)
    st = torch.zeros(1, dtype=torch.int32, device=DEV)
    ntc.ntc_decode_texels(m2, q, qo, st)
    # other profiles / depth / activation (generic instantiations), one mip each
    for name, hm, act in (("ntc0.5", 1, 0), ("ntc1.0", 1, 0), ("ntc2.25", 1, 0), ("ntc0.2", 2, 0), ("ntc0.2", 1, 1)):
        dv = Profile.named(name, 256, 16, hm, act)
        mv = material(dv, 4)
        ov = torch.empty(128 * 128 * 16, dtype=torch.float16, device=DEV)
        ntc.ntc_decode_mip(mv, 1, ov)
    # multi-material (3 materials, interleaved queries) and filtering
    mats = [material(d2, 10 + i) for i in range(3)]
    qm = ntc.pack_queries(torch.from_numpy(gen_queries(5, W, 3001).astype(np.int64)), torch.arange(3001) % 3).to(DEV)
    om = torch.empty(3001 * 9, dtype=torch.float16, device=DEV)
    ntc.ntc_decode_texels_multi(mats, qm, om)
    uvl = torch.rand(2048, 3, device=DEV)
    uvl[:, 2] *= ntc.ntc_num_mips(d2) - 1
    of = torch.empty(2048 * 9, dtype=torch.float16, device=DEV)
    for mode in range(5):
        ntc.ntc_filter_texels(m2, uvl, mode, of, seed=9)
    torch.cuda.synchronize()
    print("decode runs ok, status word", int(st.item()))


def train_runs(small):
    for name, hm, W in (("ntc0.2", 1, 512 if small else 1024), ("ntc0.2", 2, 256), ("ntc1.0", 1, 256)):
        d = Profile.named(name, W, 9, hm)
        NL, P = ntc.ntc_num_latents(d), ntc.ntc_num_params(d)
        t = {k: torch.zeros(NL, device=DEV) for k in ("m_lat", "v_lat", "grad_lat", "noisy")}
        t.update({k: torch.zeros(P, device=DEV) for k in ("m_par", "v_par", "grad_par")})
        t["latents"] = torch.from_numpy(gen_latents(1, NL)).to(DEV)
        t["params"] = torch.from_numpy(gen_weights_f32(2, d.input_dim, 9, hm)).to(DEV)
        ref = [torch.from_numpy(u8_to_f16_bits(x).view(np.int16)).to(DEV)
               for x in box_mip_chain_u8(gen_reference_u8(3, W, 9))]
        tr, bufs, loss = ntc.Trainer(d), ntc.make_buffers(t), torch.zeros(1, device=DEV)
        st = torch.zeros(1, dtype=torch.int32, device=DEV)
        for s, mip in enumerate((0, 1, 3)):
            crops = gen_crops(20 + s, W, mip, 4, 64 if small else 128)
            b = ntc.make_batch(mip, crops, ref[mip], (W >> mip) * 9)
            hp = ntc.Hparams(0.01, 0.005, 0.9, 0.999, 1e-8, s + 1, 7, 1, 0, 0)
            ntc.ntc_train_step(tr, bufs, b, hp, loss, st)
            ntc.ntc_train_step(tr, bufs, b, hp, loss, st, flags=ntc.NTC_STEP_GRADS)
            ntc.ntc_train_step(tr, bufs, b, hp, loss, st, flags=ntc.NTC_STEP_APPLY)
        torch.cuda.synchronize()
        print(f"train runs ok ({name}, depth {hm}): loss {loss.item():.5f}, status {int(st.item())}")


if __name__ == "__main__":
    small = "--small" in sys.argv
    decode_runs(small)
    train_runs(small)
