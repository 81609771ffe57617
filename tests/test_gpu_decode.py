"""GPU parity of the decode path (a0..a7) against the CPU oracle, through the C ABI.

Bars (BASELINE.json north_star): bit-exact addressing, quantised codes and assembled fp16
inputs; max abs error <= 2e-3 on decoded channels in [0, 1].
"""
import numpy as np
import pytest
import torch

import paper_2305_17105_b200 as ntc
from paper_2305_17105_b200.synth import Profile, gen_latents, gen_queries
from helpers import chain_queries, material_inputs

pytestmark = pytest.mark.gpu
TOL = 2e-3
DEV = "cuda:0"


def _material(O, d, seed, out_gain=0.3):
    codes, w = material_inputs(O, d, seed, out_gain)
    mat = ntc.Material(d, torch.from_numpy(codes).to(DEV), torch.from_numpy(w.view(np.int16)).to(DEV))
    return mat, codes, w


def _decode_queries_gpu(mat, xym):
    q = ntc.pack_queries(torch.from_numpy(xym).to(DEV))
    out = torch.empty((xym.shape[0], mat.desc.channels), dtype=torch.float16, device=DEV)
    st = torch.zeros(1, dtype=torch.int32, device=DEV)
    ntc.ntc_decode_texels(mat, q, out, st)
    torch.cuda.synchronize()
    return out.float().cpu().numpy(), int(st.item())


@pytest.mark.parametrize("name", ["ntc0.2", "ntc0.5", "ntc1.0", "ntc2.25"])
def test_quantize_bit_exact(O, name):
    """a0: codes bit-exact, including exact ties at every bin edge and out-of-range values."""
    d = Profile.named(name, 256, 8)
    n = O.num_latents(d)
    lat = gen_latents(5, n, scale=0.7)
    # plant exact ties (bin edges (idx + 1/2) Q) in both grids' bit depths
    rng = np.random.default_rng(0)
    for B in {d.b0, d.b1}:
        N = 2**B
        idx = rng.choice(n, 2000, replace=False)
        lat[idx] = ((rng.integers(-N // 2, N // 2 + 1, idx.size) + 0.5) / N).astype(np.float32)
    want = O.quantize_latents(d, lat)
    codes = torch.empty(n, dtype=torch.uint8, device=DEV)
    ntc.ntc_quantize_latents(d, torch.from_numpy(lat).to(DEV), codes)
    assert np.array_equal(codes.cpu().numpy(), want)


@pytest.mark.parametrize("name", ["ntc0.2", "ntc0.5", "ntc1.0", "ntc2.25"])
def test_assemble_bit_exact(O, name):
    """a1-a4: addressing and the fp16 input vector X bit-exact vs the oracle, every mip."""
    W = 128
    d = Profile.named(name, W, 8)
    mat, codes, _ = _material(O, d, 21)
    xym = chain_queries(W, range(O.num_mips(W)), stride=1)
    xym = xym[np.random.default_rng(1).permutation(xym.shape[0])[:6000]]
    q = ntc.pack_queries(torch.from_numpy(xym).to(DEV))
    n = xym.shape[0]
    addr = torch.empty((n, 17), dtype=torch.int32, device=DEV)
    X = torch.empty((n, d.input_dim), dtype=torch.int16, device=DEV)
    ntc.ntc_debug_assemble(mat, q, addr, X)
    addr, X = addr.cpu().numpy(), X.cpu().numpy().view(np.uint16)
    for i in range(n):
        x, y, m = xym[i]
        ti, _ = O.address(d, m, x, y)
        assert np.array_equal(addr[i], ti), (x, y, m)
        assert np.array_equal(X[i], O.assemble(d, codes, m, x, y)), (x, y, m)


def test_decode_mip_c1(O):
    """configs[0]: 256^2, 8 channels, mip 0, NTC 0.2, [57, 64, 64, 8]: every texel."""
    d = Profile.named("ntc0.2", 256, 8)
    mat, codes, w = _material(O, d, 0x4E544300)
    out = torch.empty((256, 256, 8), dtype=torch.float16, device=DEV)
    ntc.ntc_decode_mip(mat, 0, out)
    torch.cuda.synchronize()
    ref = O.decode_mip(d, codes, w, 0)
    err = np.abs(out.float().cpu().numpy() - ref)
    assert err.max() <= TOL, err.max()


@pytest.mark.parametrize("name,hm,c", [("ntc0.2", 1, 9), ("ntc0.2", 2, 9), ("ntc0.5", 1, 16), ("ntc1.0", 1, 3),
                                        ("ntc2.25", 1, 12), ("ntc2.25", 2, 16)])
def test_decode_chain_profiles(O, name, hm, c):
    """Full chain (all mips incl. ragged tail tiles) for every compiled profile / depth."""
    W = 128
    d = Profile.named(name, W, c, hm)
    mat, codes, w = _material(O, d, 7 + hm)
    T = ntc.ntc_chain_texels(d)
    out = torch.full((T * c,), float("nan"), dtype=torch.float16, device=DEV)
    ntc.ntc_decode_chain(mat, out)
    torch.cuda.synchronize()
    got = out.float().cpu().numpy()
    for m in range(O.num_mips(W)):
        wm = W >> m
        off = ntc.ntc_mip_offset(d, m) * c
        ref = O.decode_mip(d, codes, w, m).reshape(-1)
        err = np.abs(got[off: off + wm * wm * c] - ref)
        assert err.max() <= TOL, (m, err.max())


def test_decode_chain_c2_full(O):
    """configs[1]: 2048^2, 9 channels, full chain (5,592,405 texels): every texel."""
    d = Profile.named("ntc0.2", 2048, 9)
    mat, codes, w = _material(O, d, 0x4E544301)
    T = ntc.ntc_chain_texels(d)
    assert T == 5_592_405
    out = torch.empty((T * 9,), dtype=torch.float16, device=DEV)
    ntc.ntc_decode_chain(mat, out)
    torch.cuda.synchronize()
    got = out.float().cpu().numpy()
    for m in range(O.num_mips(2048)):
        wm = 2048 >> m
        off = ntc.ntc_mip_offset(d, m) * 9
        ref = O.decode_mip(d, codes, w, m).reshape(-1)
        err = np.abs(got[off: off + wm * wm * 9] - ref)
        assert err.max() <= TOL, (m, err.max())


def test_decode_stress_gain(O):
    """Stress material: output gain 1.0 (about half the outputs clamped)."""
    d = Profile.named("ntc0.2", 256, 16)
    mat, codes, w = _material(O, d, 99, out_gain=1.0)
    for m in (0, 1, 4, 8):
        wm = 256 >> m
        out = torch.empty((wm, wm, 16), dtype=torch.float16, device=DEV)
        ntc.ntc_decode_mip(mat, m, out)
        torch.cuda.synchronize()
        err = np.abs(out.float().cpu().numpy() - O.decode_mip(d, codes, w, m))
        assert err.max() <= TOL, (m, err.max())


def test_decode_mip_row_stride(O):
    d = Profile.named("ntc0.2", 64, 5)
    mat, codes, w = _material(O, d, 3)
    buf = torch.full((32, 200), -1.0, dtype=torch.float16, device=DEV)
    ntc.ntc_decode_mip(mat, 1, buf, row_stride_elems=200)
    torch.cuda.synchronize()
    got = buf.float().cpu().numpy()
    assert np.all(got[:, 160:] == -1.0)
    err = np.abs(got[:, :160].reshape(32, 32, 5) - O.decode_mip(d, codes, w, 1))
    assert err.max() <= TOL


def test_decode_texels_random_and_errors(O):
    """configs[2]-style random access (area-uniform mips, random order), an empty batch,
    and out-of-range queries (status bit + NaN row, the rest decoded normally)."""
    d = Profile.named("ntc0.2", 512, 16)
    mat, codes, w = _material(O, d, 0x4E544302)
    xym = gen_queries(5, 512, 20000, "area")
    xym2 = gen_queries(6, 512, 5000, "mip")
    allq = np.concatenate([xym, xym2])
    bad = np.array([[512, 0, 0], [0, 300, 1], [0, 0, 10], [3, 3, 40]], np.int32)
    allq = np.concatenate([allq[:100], bad, allq[100:]])
    got, st = _decode_queries_gpu(mat, allq)
    assert st & ntc.NTC_ERR_OUT_OF_RANGE
    assert np.all(np.isnan(got[100:104]))
    ok = np.ones(allq.shape[0], bool)
    ok[100:104] = False
    ref = O.decode_texels(d, codes, w, allq[ok])
    assert np.abs(got[ok] - ref).max() <= TOL
    # empty batch is a no-op
    empty = torch.empty(0, dtype=torch.int64, device=DEV)
    ntc.ntc_decode_texels(mat, empty, torch.empty((0, 16), dtype=torch.float16, device=DEV))


@pytest.mark.parametrize("c,off", [(1, 2), (3, 2), (7, 2), (9, 2), (15, 2), (9, 1)])
def test_decode_texels_odd_channels_paired_stores(O, c, off):
    """Odd c: full tiles take the paired-row store path (the even row's lane completes its
    last word with the odd row's first channel).  Bad queries on even and odd rows inside
    full tiles, a ragged tail, and the output's neighbours left untouched."""
    d = Profile.named("ntc0.2", 256, c)
    mat, codes, w = _material(O, d, 0x4E5400 + c)
    allq = gen_queries(11 + c, 256, 128 * 5 + 77, "area")
    bad_rows = [130, 131, 256 + 7, 384 + 64]
    allq[bad_rows] = np.array([[256, 0, 0], [0, 0, 9], [0, 200, 1], [5, 5, 30]], np.int32)
    n = allq.shape[0]
    q = ntc.pack_queries(torch.from_numpy(allq).to(DEV))
    buf = torch.full((n + 4, c), -1.0, dtype=torch.float16, device=DEV)
    st = torch.zeros(1, dtype=torch.int32, device=DEV)
    ntc.ntc_decode_texels(mat, q, buf[off:n + off], st)  # off = 1: 2-byte-aligned output (fallback)
    torch.cuda.synchronize()
    got = buf.float().cpu().numpy()
    assert np.all(got[:off] == -1.0) and np.all(got[n + off:] == -1.0)
    got = got[off:n + off]
    assert int(st.item()) & ntc.NTC_ERR_OUT_OF_RANGE
    ok = np.ones(n, bool)
    ok[bad_rows] = False
    assert np.all(np.isnan(got[~ok]))
    ref = O.decode_texels(d, codes, w, allq[ok])
    assert np.abs(got[ok] - ref).max() <= TOL


@pytest.mark.parametrize("stride_pad", [0, 1, 2])
def test_decode_mip_odd_channels_strides(O, stride_pad):
    """decode_mip of a 256-wide mip with odd c: even strides use the paired stores, an odd
    stride (or odd base offset) falls back to per-channel stores; padding stays untouched."""
    c = 7
    d = Profile.named("ntc0.2", 256, c)
    mat, codes, w = _material(O, d, 9)
    rs = 256 * c + stride_pad
    buf = torch.full((256 * rs + 1,), -1.0, dtype=torch.float16, device=DEV)
    view = buf[1:] if stride_pad == 2 else buf[:-1]  # odd base offset in one case
    ntc.ntc_decode_mip(mat, 0, view, row_stride_elems=rs)
    torch.cuda.synchronize()
    got = view.float().cpu().numpy().reshape(256, rs)
    assert np.all(got[:, 256 * c:] == -1.0)
    err = np.abs(got[:, :256 * c].reshape(256, 256, c) - O.decode_mip(d, codes, w, 0))
    assert err.max() <= TOL


def test_invalid_arguments(O):
    d = Profile.named("ntc0.2", 64, 8)
    mat, _, _ = _material(O, d, 1)
    out = torch.empty((64 * 64 * 8,), dtype=torch.float16, device=DEV)
    with pytest.raises(ntc.NtcError) as e:
        ntc.ntc_decode_mip(mat, 7, out)
    assert e.value.status == ntc.NTC_ERR_INVALID_ARGUMENT
    with pytest.raises(ntc.NtcError) as e:
        ntc.ntc_decode_mip(mat, 0, out, row_stride_elems=10)
    bad = Profile(64, 8, 4, 6, 3, 12, 4)
    with pytest.raises(ntc.NtcError) as e:
        ntc.Material(bad, torch.zeros(10, dtype=torch.uint8, device=DEV), torch.zeros(10, dtype=torch.int16, device=DEV))
    assert e.value.status == ntc.NTC_ERR_UNSUPPORTED


def test_smallest_texture(O):
    """W = 8 (one feature level, G0 2x2, G1 1x1): the degenerate geometry."""
    d = Profile.named("ntc0.2", 8, 4)
    mat, codes, w = _material(O, d, 2)
    T = ntc.ntc_chain_texels(d)
    out = torch.empty((T * 4,), dtype=torch.float16, device=DEV)
    ntc.ntc_decode_chain(mat, out)
    torch.cuda.synchronize()
    got = out.float().cpu().numpy()
    ref = np.concatenate([O.decode_mip(d, codes, w, m).reshape(-1) for m in range(4)])
    assert np.abs(got - ref).max() <= TOL


def test_full_size_4k_sampled(O):
    """configs[2] at full size in the bench launch configuration: 4096^2, 16 ch chain
    decoded by one ntc_decode_chain launch; 200k sampled texels (all mips) vs the oracle."""
    d = Profile.named("ntc0.2", 4096, 16)
    mat, codes, w = _material(O, d, 0x4E544302)
    T = ntc.ntc_chain_texels(d)
    out = torch.empty((T * 16,), dtype=torch.float16, device=DEV)
    ntc.ntc_decode_chain(mat, out)
    torch.cuda.synchronize()
    xym = gen_queries(11, 4096, 200000, "mip")
    offs = np.array([ntc.ntc_mip_offset(d, m) for m in range(13)], np.int64)
    idx = offs[xym[:, 2]] + xym[:, 1].astype(np.int64) * (4096 >> xym[:, 2]) + xym[:, 0]
    got = out.view(-1, 16)[torch.from_numpy(idx).to(DEV)].float().cpu().numpy()
    ref = O.decode_texels(d, codes, w, xym)
    assert np.abs(got - ref).max() <= TOL


@pytest.mark.parametrize("name,hm,c", [("ntc0.2", 1, 9), ("ntc0.2", 2, 8), ("ntc0.5", 1, 16), ("ntc2.25", 2, 12)])
def test_decode_gelu_variant(O, name, hm, c):
    """f4: exact GELU activation (activation = 1) -- full chain and random
    queries vs the oracle, every compiled profile family, both depths."""
    W = 128
    d = Profile.named(name, W, c, hm, activation=1)
    mat, codes, w = _material(O, d, 61 + hm)
    T = ntc.ntc_chain_texels(d)
    out = torch.full((T * c,), float("nan"), dtype=torch.float16, device=DEV)
    ntc.ntc_decode_chain(mat, out)
    torch.cuda.synchronize()
    got = out.float().cpu().numpy()
    for m in range(O.num_mips(W)):
        wm = W >> m
        off = ntc.ntc_mip_offset(d, m) * c
        err = np.abs(got[off: off + wm * wm * c] - O.decode_mip(d, codes, w, m).reshape(-1))
        assert err.max() <= TOL, (m, err.max())
    xym = gen_queries(5, W, 5000)
    gq, st = _decode_queries_gpu(mat, xym)
    assert st == 0
    assert np.abs(gq - O.decode_texels(d, codes, w, xym)).max() <= TOL


def test_bench_configs_sampled(O):
    """The bench's own launch configurations at full size (bench.py): the 4096^2 9-ch chain
    material of the headline line (seed base + 4) through one ntc_decode_chain launch, and the
    `random` line's 2^24 area-uniform queries on the 4096^2 16-ch material through one
    ntc_decode_texels launch; sampled rows vs the oracle."""
    from paper_2305_17105_b200.synth import SEED_BASE, gen_codes, gen_weights_f16

    rng = np.random.default_rng(123)
    # headline: decode chain
    d = Profile.named("ntc0.2", 4096, 9)
    codes = gen_codes(SEED_BASE + 4, ntc.grid_list(d))
    w = gen_weights_f16(SEED_BASE + 5, d.input_dim, 9)
    mat = ntc.Material(d, torch.from_numpy(codes).to(DEV), torch.from_numpy(w.view(np.int16)).to(DEV))
    T = ntc.ntc_chain_texels(d)
    out = torch.empty((T, 9), dtype=torch.float16, device=DEV)
    ntc.ntc_decode_chain(mat, out)
    torch.cuda.synchronize()
    xym = gen_queries(21, 4096, 150000, "mip")
    offs = np.array([ntc.ntc_mip_offset(d, m) for m in range(13)], np.int64)
    idx = offs[xym[:, 2]] + xym[:, 1].astype(np.int64) * (4096 >> xym[:, 2]) + xym[:, 0]
    got = out[torch.from_numpy(idx).to(DEV)].float().cpu().numpy()
    assert np.abs(got - O.decode_texels(d, codes, w, xym)).max() <= TOL
    del out, mat
    # random line: 2^24 queries, 16 channels
    d = Profile.named("ntc0.2", 4096, 16)
    codes = gen_codes(SEED_BASE + 2, ntc.grid_list(d))
    w = gen_weights_f16(SEED_BASE + 3, d.input_dim, 16)
    mat = ntc.Material(d, torch.from_numpy(codes).to(DEV), torch.from_numpy(w.view(np.int16)).to(DEV))
    n = 1 << 24
    xym = gen_queries(SEED_BASE + 4, 4096, n, "area")
    out = torch.empty((n, 16), dtype=torch.float16, device=DEV)
    st = torch.zeros(1, dtype=torch.int32, device=DEV)
    ntc.ntc_decode_texels(mat, ntc.pack_queries(torch.from_numpy(xym).to(DEV)), out, st)
    torch.cuda.synchronize()
    assert st.item() == 0
    sel = rng.choice(n, 150000, replace=False)
    got = out[torch.from_numpy(sel).to(DEV)].float().cpu().numpy()
    assert np.abs(got - O.decode_texels(d, codes, w, xym[sel])).max() <= TOL


@pytest.mark.parametrize("off", [0, 1, 8])
def test_decode_texels_c16_alignment(O, off):
    """c = 16 (the random-access line's compiled instantiation): 16-byte vector stores when the
    output rows are 16-byte aligned, per-word stores otherwise; neighbours left untouched."""
    d = Profile.named("ntc0.2", 256, 16)
    mat, codes, w = _material(O, d, 0x4E5416)
    allq = gen_queries(31, 256, 128 * 3 + 50, "area")
    n = allq.shape[0]
    q = ntc.pack_queries(torch.from_numpy(allq).to(DEV))
    buf = torch.full((n * 16 + 32,), -1.0, dtype=torch.float16, device=DEV)
    ntc.ntc_decode_texels(mat, q, buf[off:off + n * 16])
    torch.cuda.synchronize()
    got = buf.float().cpu().numpy()
    assert np.all(got[:off] == -1.0) and np.all(got[off + n * 16:] == -1.0)
    ref = O.decode_texels(d, codes, w, allq)
    assert np.abs(got[off:off + n * 16].reshape(n, 16) - ref).max() <= TOL


def test_maximum_texture_size(O):
    """The largest texture the ABI accepts, 32768^2 (16 mips; NTC 0.2 level 0 alone holds
    8192^2 x 8 G0 codes): random queries over every mip including the far corners (x, y =
    32767 in the 16-bit query fields) and a whole mid mip, against the oracle."""
    d = Profile.named("ntc0.2", 32768, 2)
    mat, codes, w = _material(O, d, 0x4E5432)
    q = gen_queries(91, 32768, 6000, "mip")
    M = 16
    corners = np.array([[(32768 >> m) - 1, (32768 >> m) - 1, m] for m in range(M)] +
                       [[0, (32768 >> m) - 1, m] for m in range(M)], np.int32)
    q = np.concatenate([q, corners])
    got, st = _decode_queries_gpu(mat, q)
    assert st == 0
    ref = O.decode_texels(d, codes, w, q)
    assert np.abs(got - ref).max() <= TOL
    out = torch.empty((256 * 256 * 2,), dtype=torch.float16, device=DEV)
    ntc.ntc_decode_mip(mat, 7, out)  # 256^2
    torch.cuda.synchronize()
    err = np.abs(out.float().cpu().numpy().reshape(256, 256, 2) - O.decode_mip(d, codes, w, 7))
    assert err.max() <= TOL
