"""Three random-access decode launches (configs[2]: 2^24 area-uniform queries, 4096^2 x 16ch),
for an ncu capture of the query kernel (profiling helper, not product code)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2305_17105_b200 as ntc  # noqa: E402
from paper_2305_17105_b200.synth import SEED_BASE, Profile, gen_codes, gen_queries, gen_weights_f16  # noqa: E402

dev = torch.device("cuda", 0)
d = Profile.named("ntc0.2", 4096, 16)
mat = ntc.Material(d, torch.from_numpy(gen_codes(SEED_BASE + 2, ntc.grid_list(d))).to(dev),
                   torch.from_numpy(gen_weights_f16(SEED_BASE + 3, d.input_dim, 16).view(np.int16)).to(dev))
n = 1 << 24
q = ntc.pack_queries(torch.from_numpy(gen_queries(SEED_BASE + 4, 4096, n, "area")).to(dev))
out = torch.empty((n, 16), dtype=torch.float16, device=dev)
for _ in range(3):
    ntc.ntc_decode_texels(mat, q, out)
torch.cuda.synchronize()
