"""Full compression of one 4096^2 9-channel material with the paper's schedule (f1,
profiling helper, not product code): 250,000 noisy steps of 8 x 256^2 crops (PAPER.md:510,
571), explicit quantisation, 5% frozen weight-only finetune; then decode the
compressed material and report the wall time, the device time of the training steps and the
PSNR of mip 0 against the (synthetic) reference.  The paper's number for this job: 1-15 min
on an RTX 4090.

usage: python tools/measure_compression.py [steps] [OUT.json]"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2305_17105_b200 as ntc  # noqa: E402
from paper_2305_17105_b200.compress import CompressConfig, Compressor  # noqa: E402
from paper_2305_17105_b200.synth import (SEED_BASE, Profile, box_mip_chain_u8, gen_reference_u8,  # noqa: E402
                                         u8_to_f16_bits)


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 250_000
    out_path = sys.argv[2] if len(sys.argv) > 2 else None
    dev = "cuda:0"
    W, C = 4096, 9
    d = Profile.named("ntc0.2", W, C)
    chain = [torch.from_numpy(u8_to_f16_bits(m).view(np.int16).copy()).to(dev)
             for m in box_mip_chain_u8(gen_reference_u8(SEED_BASE + 3, W, C))]
    cfg = CompressConfig(steps=steps, seed=7)
    comp = Compressor(d, chain, cfg, dev)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    codes, w16 = comp.run(log_every=max(1, steps // 20))
    e1.record()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    # decode mip 0 of the compressed material, PSNR against the reference
    mat = ntc.Material(d, codes, w16.view(torch.int16))
    out = torch.empty((W, W, C), dtype=torch.float16, device=dev)
    ntc.ntc_decode_mip(mat, 0, out)
    ref = chain[0].view(torch.float16).float().view(W, W, C)
    mse = torch.mean((out.float() - ref) ** 2).item()
    res = {"workload": f"4096^2 x {C}ch NTC0.2, {steps} noisy steps + {comp.total - steps} frozen steps, "
                       f"{cfg.crops} x {cfg.crop}^2 crops, LOD law + cosine LR (f1)",
           "steps_total": comp.total, "wall_s": round(wall, 2), "device_s": round(e0.elapsed_time(e1) / 1e3, 2),
           "ms_per_step": round(e0.elapsed_time(e1) / comp.total, 4), "psnr_mip0_db": round(-10 * np.log10(mse), 2),
           "loss_first_last": [comp.losses[0][1], comp.losses[-1][1]] if comp.losses else None,
           "paper": "1-15 min per 4k 9-channel set on an RTX 4090 (PAPER.md:199)"}
    print(json.dumps(res), flush=True)
    if out_path:
        with open(out_path, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
