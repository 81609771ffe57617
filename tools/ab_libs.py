"""A/B timing between library builds (profiling helper, not product code):
  python tools/ab_decode.py [--train] LIB_A.so LIB_B.so [...] [--rounds R]
alternates the builds in separate processes (one library per process), L2 flushed before each
run, CUDA events: the headline chain decodes (c = 9, 16), or with --train the C4 step, --random
the configs[2] random queries, --profiles the other Table 2 profiles and depth B."""
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


CHILD_TRAIN = r'''
import sys, json, numpy as np, torch
sys.path.insert(0, %r)
import paper_2305_17105_b200 as ntc
ntc.LIB_PATH = %r
from bench import _device_time
from paper_2305_17105_b200.synth import (SEED_BASE, Profile, gen_crops, gen_latents, gen_reference_u8,
                                         gen_weights_f32, u8_to_f16_bits)
dev = torch.device("cuda", 0)
d = Profile.named("ntc0.2", 4096, 9)
NL, P = ntc.ntc_num_latents(d), ntc.ntc_num_params(d)
t = {k: torch.zeros(NL, device=dev) for k in ("m_lat", "v_lat", "grad_lat", "noisy")}
t.update({k: torch.zeros(P, device=dev) for k in ("m_par", "v_par", "grad_par")})
t["latents"] = torch.from_numpy(gen_latents(SEED_BASE + 6, NL)).to(dev)
t["params"] = torch.from_numpy(gen_weights_f32(SEED_BASE + 7, d.input_dim, 9)).to(dev)
ref = torch.from_numpy(u8_to_f16_bits(gen_reference_u8(SEED_BASE + 4, 1024, 9)).view(np.int16)).to(dev)
ref = ref.reshape(1024, 1024 * 9).repeat(4, 4).reshape(-1).contiguous()
tr, bufs, loss = ntc.Trainer(d), ntc.make_buffers(t), torch.zeros(1, device=dev)
crops = gen_crops(SEED_BASE + 3, 4096, 0, 4, 256)
st = [0]
def run():
    st[0] += 1
    ntc.ntc_train_step(tr, bufs, ntc.make_batch(0, crops, ref, 4096 * 9),
                       ntc.Hparams(0.01, 0.005, 0.9, 0.999, 1e-8, st[0], 7, 1, 0), loss)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
print(json.dumps({"train_us": _device_time(torch, run, flush, 50) * 1e6}))
'''


CHILD_RANDOM = r'''
import sys, json, numpy as np, torch
sys.path.insert(0, %r)
import paper_2305_17105_b200 as ntc
ntc.LIB_PATH = %r
from bench import _device_time
from paper_2305_17105_b200.synth import SEED_BASE, Profile, gen_codes, gen_queries, gen_weights_f16
dev = torch.device("cuda", 0)
d = Profile.named("ntc0.2", 4096, 16)
mat = ntc.Material(d, torch.from_numpy(gen_codes(SEED_BASE + 2, ntc.grid_list(d))).to(dev),
                   torch.from_numpy(gen_weights_f16(SEED_BASE + 3, d.input_dim, 16).view(np.int16)).to(dev))
n = 1 << 24
q = ntc.pack_queries(torch.from_numpy(gen_queries(SEED_BASE + 4, 4096, n, "area")).to(dev))
out = torch.empty((n, 16), dtype=torch.float16, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
t = _device_time(torch, lambda: ntc.ntc_decode_texels(mat, q, out), flush, 20)
print(json.dumps({"random_c16": n / t / 1e9}))
'''

CHILD_PROFILES = r'''
import sys, json, numpy as np, torch
sys.path.insert(0, %r)
import paper_2305_17105_b200 as ntc
ntc.LIB_PATH = %r
from bench import _device_time
from paper_2305_17105_b200.synth import SEED_BASE, Profile, gen_codes, gen_weights_f16
dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
out = {}
for name, hm in (("ntc0.5", 1), ("ntc1.0", 1), ("ntc2.25", 1), ("ntc0.2", 2)):
    d = Profile.named(name, 4096, 9, hm)
    mat = ntc.Material(d, torch.from_numpy(gen_codes(SEED_BASE + 4, ntc.grid_list(d))).to(dev),
                       torch.from_numpy(gen_weights_f16(SEED_BASE + 5, d.input_dim, 9, hm).view(np.int16)).to(dev))
    T = ntc.ntc_chain_texels(d)
    o = torch.empty(T * 9, dtype=torch.float16, device=dev)
    t = _device_time(torch, lambda: ntc.ntc_decode_chain(mat, o), flush, 10)
    out[name + ("" if hm == 1 else "_B")] = T / t / 1e9
print(json.dumps(out))
'''


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    rounds = int(sys.argv[sys.argv.index("--rounds") + 1]) if "--rounds" in sys.argv else 3
    child = CHILD_TRAIN if "--train" in sys.argv else (CHILD_RANDOM if "--random" in sys.argv else CHILD)
    if "--profiles" in sys.argv:
        child = CHILD_PROFILES
    libs = [a for a in args if a.endswith(".so")]
    res = {l: [] for l in libs}
    for _ in range(rounds):
        for l in libs:
            r = subprocess.run([sys.executable, "-c", child % (ROOT, os.path.abspath(l))], capture_output=True, text=True)
            res[l].append(json.loads(r.stdout.strip().splitlines()[-1]))
    for l in libs:
        print(l, json.dumps(res[l]))


if __name__ == "__main__":
    main()
