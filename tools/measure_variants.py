"""Secondary decode rows of SURVEY.md 8(d) (profiling helper, not product code): full-chain
decode throughput of a 4096^2 9-channel material for every compiled profile, depth reading B
(hidden_mats = 2) and the exact-GELU variant, timed like bench.py (L2 flushed before each
run, CUDA events).  usage: python tools/measure_variants.py [OUT.json]"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2305_17105_b200 as ntc  # noqa: E402
from bench import _device_time, _peaks, decode_flops_per_texel  # noqa: E402
from paper_2305_17105_b200.synth import SEED_BASE, Profile, gen_codes, gen_weights_f16  # noqa: E402


def main():
    out_path = sys.argv[1] if len(sys.argv) > 1 else None
    dev = torch.device("cuda", 0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    pk, _ = _peaks()
    rows = []
    for name, hm, act in [("ntc0.2", 1, 0), ("ntc0.5", 1, 0), ("ntc1.0", 1, 0), ("ntc2.25", 1, 0),
                          ("ntc0.2", 2, 0), ("ntc0.2", 1, 1)]:
        d = Profile.named(name, 4096, 9, hm, act)
        seed = SEED_BASE + 4
        mat = ntc.Material(d, torch.from_numpy(gen_codes(seed, ntc.grid_list(d))).to(dev),
                           torch.from_numpy(gen_weights_f16(seed + 1, d.input_dim, 9, hm).view(np.int16)).to(dev))
        T = ntc.ntc_chain_texels(d)
        out = torch.empty((T * 9,), dtype=torch.float16, device=dev)
        t = _device_time(torch, lambda: ntc.ntc_decode_chain(mat, out), flush, 10)
        tf = decode_flops_per_texel(d) * T / t / 1e12
        rows.append({"profile": name, "hidden_mats": hm, "activation": ["hardGELU", "GELU"][act],
                     "D": d.input_dim, "ms": round(t * 1e3, 4), "Gtexel_s": round(T / t / 1e9, 3),
                     "tflops": round(tf, 1), "frac_tensor": round(tf / pk["bf16_tflops"], 4)})
        print(json.dumps(rows[-1]), flush=True)
        del mat, out
    # training step rows: 4 x 256^2 crops at LOD 0 of a 4096^2 9-channel material
    from bench import train_flops_per_texel  # noqa: E402
    from paper_2305_17105_b200.synth import gen_crops, gen_latents, gen_reference_u8, gen_weights_f32, u8_to_f16_bits

    trows = []
    ref = torch.from_numpy(u8_to_f16_bits(gen_reference_u8(SEED_BASE + 4, 4096, 9)).view(np.int16)).to(dev)
    for name, hm, act in [("ntc0.2", 1, 0), ("ntc0.5", 1, 0), ("ntc1.0", 1, 0), ("ntc2.25", 1, 0),
                          ("ntc0.2", 2, 0), ("ntc0.2", 1, 1)]:
        d = Profile.named(name, 4096, 9, hm, act)
        NL, P = ntc.ntc_num_latents(d), ntc.ntc_num_params(d)
        t = {k: torch.zeros(NL, device=dev) for k in ("m_lat", "v_lat", "grad_lat", "noisy")}
        t.update({k: torch.zeros(P, device=dev) for k in ("m_par", "v_par", "grad_par")})
        t["latents"] = torch.from_numpy(gen_latents(SEED_BASE + 6, NL)).to(dev)
        t["params"] = torch.from_numpy(gen_weights_f32(SEED_BASE + 7, d.input_dim, 9, hm)).to(dev)
        tr, bufs, loss = ntc.Trainer(d), ntc.make_buffers(t), torch.zeros(1, device=dev)
        crops = gen_crops(SEED_BASE + 3, 4096, 0, 4, 256)
        step = [0]

        def run():
            step[0] += 1
            ntc.ntc_train_step(tr, bufs, ntc.make_batch(0, crops, ref, 4096 * 9),
                               ntc.Hparams(0.01, 0.005, 0.9, 0.999, 1e-8, step[0], 7, 1, 0), loss)

        tt = _device_time(torch, run, flush, 20)
        B = 4 * 256 * 256
        tf = train_flops_per_texel(d) * B / tt / 1e12
        trows.append({"profile": name, "hidden_mats": hm, "activation": ["hardGELU", "GELU"][act],
                      "ms": round(tt * 1e3, 4), "G_texels_s": round(B / tt / 1e9, 3), "tflops": round(tf, 1),
                      "frac_tensor": round(tf / pk["bf16_tflops"], 4)})
        print(json.dumps(trows[-1]), flush=True)
    if out_path:
        with open(out_path, "w") as f:
            json.dump({"workload": "4096^2 x 9ch full-chain decode (22,369,621 texels), L2 flushed", "rows": rows,
                       "train_workload": "4096^2 x 9ch train step (GRADS|APPLY), 4 x 256^2 crops at LOD 0",
                       "train_rows": trows}, f, indent=1)


if __name__ == "__main__":
    main()
