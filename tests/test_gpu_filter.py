"""GPU parity of texture filtering on top of the decode (f2) vs the oracle: nearest,
bilinear, trilinear, stochastic bilinear/trilinear (same Philox jitter, so the same texels)."""
import numpy as np
import pytest
import torch

import paper_2305_17105_b200 as ntc
from paper_2305_17105_b200.synth import Profile
from helpers import material_inputs

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


@pytest.mark.parametrize("mode", [0, 1, 2, 3, 4])
def test_filter_parity(O, mode):
    d = Profile.named("ntc0.2", 256, 9)
    codes, w = material_inputs(O, d, 31)
    mat = ntc.Material(d, torch.from_numpy(codes).to(DEV), torch.from_numpy(w.view(np.int16)).to(DEV))
    rng = np.random.default_rng(mode)
    n = 20000
    uvl = np.c_[rng.random((n, 2)), rng.uniform(0, 8.9, n)].astype(np.float32)
    uvl[:50, 2] = np.floor(uvl[:50, 2])  # integer LODs
    uvl[50:60, :2] = 0.0                 # corner: clamp-to-edge taps
    out = torch.empty((n, 9), dtype=torch.float16, device=DEV)
    ntc.ntc_filter_texels(mat, torch.from_numpy(uvl).to(DEV), mode, out, seed=1234)
    torch.cuda.synchronize()
    ref = O.filter_texels(d, codes, w, uvl.astype(np.float64), mode, seed=1234)
    err = np.abs(out.float().cpu().numpy() - ref)
    assert err.max() <= 2e-3, err.max()
