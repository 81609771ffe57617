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
