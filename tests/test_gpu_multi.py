"""GPU parity of the multi-material random-access decode against the CPU
oracle, through the C ABI: every query's row must match the oracle decode of ITS material
(max abs error <= 2e-3), independent of how the library buckets and orders the queries."""
import numpy as np
import pytest
import torch

import paper_2305_17105_b200 as ntc
from paper_2305_17105_b200.synth import Profile, gen_queries
from helpers import material_inputs

pytestmark = pytest.mark.gpu
TOL = 2e-3
DEV = "cuda:0"


def _materials(O, d, seeds, out_gain=0.3):
    mats, ins = [], []
    for s in seeds:
        codes, w = material_inputs(O, d, s, out_gain)
        mats.append(ntc.Material(d, torch.from_numpy(codes).to(DEV), torch.from_numpy(w.view(np.int16)).to(DEV)))
        ins.append((codes, w))
    return mats, ins


def _run(mats, xym, mat_idx):
    q = ntc.pack_queries(torch.from_numpy(xym).to(DEV), torch.from_numpy(mat_idx).to(DEV))
    out = torch.empty((xym.shape[0], mats[0].desc.channels), dtype=torch.float16, device=DEV)
    st = torch.zeros(1, dtype=torch.int32, device=DEV)
    ntc.ntc_decode_texels_multi(mats, q, out, st)
    torch.cuda.synchronize()
    return out.float().cpu().numpy(), int(st.item())


def _check(O, d, ins, xym, mat_idx, got):
    for k, (codes, w) in enumerate(ins):
        sel = np.nonzero(mat_idx == k)[0]
        if sel.size == 0:
            continue
        ref = O.decode_texels(d, codes, w, xym[sel])
        err = np.abs(got[sel] - ref).max()
        assert err <= TOL, (k, err)


@pytest.mark.parametrize("name,hm", [("ntc0.2", 1), ("ntc0.5", 1), ("ntc0.2", 2)])
def test_multi_random_interleaved(O, name, hm):
    """5 materials, queries interleaved at random (the divergent case), ragged counts."""
    W = 256
    d = Profile.named(name, W, 9, hidden_mats=hm)
    mats, ins = _materials(O, d, [101, 202, 303, 404, 505])
    n = 20011
    xym = gen_queries(7, W, n)
    mat_idx = np.random.default_rng(3).integers(0, len(mats), n).astype(np.int32)
    got, st = _run(mats, xym, mat_idx)
    assert st == 0
    _check(O, d, ins, xym, mat_idx, got)


def test_multi_skewed_and_empty_materials(O):
    """Highly skewed material histogram, some materials with no query, one with exactly one."""
    W = 128
    d = Profile.named("ntc0.2", W, 8)
    mats, ins = _materials(O, d, [11, 12, 13, 14, 15, 16, 17])
    n = 9000
    xym = gen_queries(9, W, n)
    rng = np.random.default_rng(4)
    mat_idx = np.where(rng.random(n) < 0.9, 2, 5).astype(np.int32)  # materials 0,1,3,4,6 empty ...
    mat_idx[17] = 6                                                 # ... except one query of 6
    got, st = _run(mats, xym, mat_idx)
    assert st == 0
    _check(O, d, ins, xym, mat_idx, got)


def test_multi_equals_single_material_calls(O):
    """Each query's row equals the single-material ntc_decode_texels row bit for bit: the
    bucketing only reorders tiles, the per-texel arithmetic is the same kernel body."""
    W = 256
    d = Profile.named("ntc0.2", W, 9)
    mats, _ = _materials(O, d, [21, 22, 23])
    n = 12345
    xym = gen_queries(11, W, n)
    mat_idx = np.random.default_rng(5).integers(0, 3, n).astype(np.int32)
    got, st = _run(mats, xym, mat_idx)
    assert st == 0
    for k, mat in enumerate(mats):
        sel = np.nonzero(mat_idx == k)[0]
        q = ntc.pack_queries(torch.from_numpy(xym[sel]).to(DEV))
        out = torch.empty((sel.size, 9), dtype=torch.float16, device=DEV)
        ntc.ntc_decode_texels(mat, q, out)
        torch.cuda.synchronize()
        assert np.array_equal(out.float().cpu().numpy(), got[sel])


def test_multi_bad_material_and_texel(O):
    """Material index >= n_mats and out-of-range texels: NaN rows + NTC_ERR_OUT_OF_RANGE; the
    rest of the batch decodes normally."""
    W = 64
    d = Profile.named("ntc0.2", W, 8)
    mats, ins = _materials(O, d, [31, 32])
    n = 3000
    xym = gen_queries(13, W, n)
    mat_idx = np.random.default_rng(6).integers(0, 2, n).astype(np.int32)
    mat_idx[[5, 700, 2999]] = [2, 255, 7]  # bad material indices
    xym[[10, 11]] = [[W, 0, 0], [0, 0, 9]]  # bad texel, bad mip
    got, st = _run(mats, xym, mat_idx)
    assert st == ntc.NTC_ERR_OUT_OF_RANGE
    bad = np.zeros(n, bool)
    bad[[5, 700, 2999, 10, 11]] = True
    assert np.isnan(got[bad]).all()
    ok = ~bad
    _check(O, d, ins, xym[ok], mat_idx[ok], got[ok])


def test_multi_single_material_many_tiles(O):
    """n_mats = 1 reduces to the plain query decode (full chain of a 512^2 material)."""
    W = 512
    d = Profile.named("ntc0.2", W, 9)
    mats, ins = _materials(O, d, [41])
    xym = gen_queries(17, W, 70000)
    got, st = _run(mats, xym, np.zeros(xym.shape[0], np.int32))
    assert st == 0
    _check(O, d, ins, xym, np.zeros(xym.shape[0], np.int32), got)


def test_multi_rejects_mixed_descs(O):
    W = 64
    d1 = Profile.named("ntc0.2", W, 8)
    d2 = Profile.named("ntc0.2", W, 9)
    m1, _ = _materials(O, d1, [1])
    m2, _ = _materials(O, d2, [2])
    q = ntc.pack_queries(torch.zeros((4, 3), dtype=torch.int32, device=DEV))
    out = torch.empty((4, 9), dtype=torch.float16, device=DEV)
    with pytest.raises(RuntimeError):
        ntc.ntc_decode_texels_multi(m1 + m2, q, out)


def test_multi_bench_screen_workload_sampled(O):
    """The bench's `multi` line at full size: the Table 4 analog (8,294,400 screen-order mip-0
    queries, 8 materials of 4096^2 x 8 ch, one material per 64x64 screen block) in one
    ntc_decode_texels_multi call; sampled rows vs the oracle decode of their material."""
    import bench
    from paper_2305_17105_b200.synth import SEED_BASE, gen_codes, gen_weights_f16

    d = Profile.named("ntc0.2", 4096, 8)
    mats, ins = [], []
    for k in range(8):
        codes = gen_codes(SEED_BASE + 4 + k, ntc.grid_list(d))
        w = gen_weights_f16(SEED_BASE + 5 + k, d.input_dim, 8)
        mats.append(ntc.Material(d, torch.from_numpy(codes).to(DEV), torch.from_numpy(w.view(np.int16)).to(DEV)))
        ins.append((codes, w))
    xym, mid = bench.screen_queries(8)
    got_all, st = _run(mats, xym, mid)
    assert st == 0
    sel = np.random.default_rng(7).choice(xym.shape[0], 80000, replace=False)
    _check(O, d, ins, xym[sel], mid[sel], got_all[sel])
