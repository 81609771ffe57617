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
    if out_path:
        with open(out_path, "w") as f:
            json.dump({"workload": "4096^2 x 9ch full-chain decode (22,369,621 texels), L2 flushed", "rows": rows},
                      f, indent=1)


if __name__ == "__main__":
    main()
