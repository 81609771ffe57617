"""A/B timing of the headline chain decode between library builds (profiling helper, not
product code): python tools/ab_decode.py LIB_A.so LIB_B.so [rounds]  -- alternates the builds in
separate processes (one library per process), L2 flushed before each run, CUDA events."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import sys, json, numpy as np, torch
sys.path.insert(0, %r)
import paper_2305_17105_b200 as ntc
ntc.LIB_PATH = %r
from bench import _device_time
from paper_2305_17105_b200.synth import SEED_BASE, Profile, gen_codes, gen_weights_f16
dev = torch.device("cuda", 0)
out = {}
for c in (9, 16):
    d = Profile.named("ntc0.2", 4096, c)
    mat = ntc.Material(d, torch.from_numpy(gen_codes(SEED_BASE + 4, ntc.grid_list(d))).to(dev),
                       torch.from_numpy(gen_weights_f16(SEED_BASE + 5, d.input_dim, c).view(np.int16)).to(dev))
    T = ntc.ntc_chain_texels(d)
    o = torch.empty(T * c, dtype=torch.float16, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    t = _device_time(torch, lambda: ntc.ntc_decode_chain(mat, o), flush, 20)
    out["c%%d" %% c] = T / t / 1e9
print(json.dumps(out))
'''


def main():
    libs = sys.argv[1:3]
    rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    res = {l: [] for l in libs}
    for _ in range(rounds):
        for l in libs:
            r = subprocess.run([sys.executable, "-c", CHILD % (ROOT, os.path.abspath(l))], capture_output=True, text=True)
            res[l].append(json.loads(r.stdout.strip().splitlines()[-1]))
    for l in libs:
        print(l, json.dumps(res[l]))


if __name__ == "__main__":
    main()
