"""Oracle pins: level mapping, grid geometry and addressing (CPU only).

Pinned against values the paper prints (Table 1, Table 2, Appendix D), SPEC.md
examples, an integer re-derivation of the tap indices, and torch's grid_sample
(texel-centre bilinear with border clamping) as an independent library routine.
"""
import numpy as np
import pytest
import torch

from conftest import golden
from paper_2305_17105_b200.synth import PROFILES, Profile, gen_codes


def test_table1_1024(O):
    """levels, G0/G1 resolutions and mip groups for 1024^2."""
    d = Profile.named("ntc0.2", 1024, 9)
    rows = golden("table1_1024.txt")
    assert O.num_levels(d) == len(rows)
    assert O.num_mips(1024) == 11
    for j, r0, r1, mips in rows:
        assert O.grid_res(d, int(j)) == (int(r0), int(r1))
        for m in map(int, mips.split(",")):
            assert O.level_of_mip(d, m) == int(j)


def test_table2_g00_resolution(O):
    """G^0_0 resolution per profile at 4096^2."""
    for name, res, c0, b0, c1, b1 in golden("table2_profiles.txt"):
        assert PROFILES[name][1:] == (int(c0), int(b0), int(c1), int(b1))
        d = Profile.named(name, 4096, 9)
        assert O.grid_res(d, 0)[0] == int(res)
        assert O.grid_res(d, 0)[1] == int(res) // 2


def test_spec_level_examples(O):
    """SPEC.md:115-118 and the 'bottom three mips' statement at 4096^2."""
    d11 = Profile.named("ntc0.2", 1024, 9)
    assert O.level_of_mip(d11, 5) == 1
    assert O.level_of_mip(d11, 9) == 3
    assert O.level_of_mip(d11, 0) == 0
    d13 = Profile.named("ntc0.2", 4096, 9)
    assert O.num_mips(4096) == 13
    L = O.num_levels(d13)
    assert [m for m in range(13) if O.level_of_mip(d13, m) == L - 1] == [10, 11, 12]
    assert O.level_of_mip(d13, 12) == 4
    # SPEC.md:118 "(mip 12, 13 mips) -> level 4" holds for every profile, the ratio-2 ones
    # (NTC 1.0 / 2.25, G^0_0 = W/2) included: their G1 could shrink once more, but "the last
    # feature level represents the bottom three mip levels"
    for name in PROFILES:
        d = Profile.named(name, 4096, 9)
        assert O.num_levels(d) == 5
        assert [O.level_of_mip(d, m) for m in range(13)] == [0, 0, 0, 0, 1, 1, 2, 2, 3, 3, 4, 4, 4]
        # ... and the Table 1 grouping at 1024^2
        d = Profile.named(name, 1024, 9)
        assert [O.level_of_mip(d, m) for m in range(11)] == [0, 0, 0, 0, 1, 1, 2, 2, 3, 3, 3]
    # every level but the first and the last serves exactly two mips, the last two or three
    # (PAPER.md:396), for every profile and size
    for name in PROFILES:
        for W in (16, 32, 64, 128, 256, 512, 1024, 2048, 4096, 8192):
            d = Profile.named(name, W, 8)
            L = O.num_levels(d)
            groups = [[m for m in range(O.num_mips(W)) if O.level_of_mip(d, m) == j] for j in range(L)]
            if L > 1:
                assert groups[0] == [0, 1, 2, 3]
                assert all(len(g) == 2 for g in groups[1:-1])
                assert len(groups[-1]) in (2, 3)
            assert sorted(sum(groups, [])) == list(range(O.num_mips(W)))
            # G1 of the last level is at least 1x1 ("cannot be further downsampled")
            assert O.grid_res(d, L - 1)[1] >= 1 and O.grid_res(d, L - 1)[0] >= 2


def test_spec_geometry_examples(O):
    """SPEC.md:125-128."""
    assert O.grid_res(Profile.named("ntc0.2", 1024, 9), 0) == (256, 128)
    assert O.grid_res(Profile.named("ntc0.2", 1024, 9), 2) == (16, 8)
    assert O.grid_res(Profile.named("ntc1.0", 4096, 9), 0) == (2048, 1024)
    assert O.grid_res(Profile.named("ntc0.2", 8192, 9), 1) == (512, 256)


def _grid_bits(O, d, levels):
    bits = 0
    for j in levels:
        r0, r1 = O.grid_res(d, j)
        bits += r0 * r0 * d.c0 * d.b0 + r1 * r1 * d.c1 * d.b1
    return bits


def test_appendix_d_storage(O):
    """Grids (MB) row; 2k/4k = level 0 exactly, 8k = pyramid (<0.02%)."""
    for name, res, mb, scope in golden("appendixD_storage.txt"):
        d = Profile.named(name, int(res), 9)
        L = O.num_levels(d)
        levels = [0] if scope == "level0" else list(range(L))
        mib = _grid_bits(O, d, levels) / 8 / 2**20
        if scope == "level0":
            assert mib == float(mb)
        else:
            assert abs(mib - float(mb)) / float(mb) < 2e-4


def test_latent_layout_offsets(O):
    d = Profile.named("ntc0.2", 256, 8)
    L = O.num_levels(d)
    off = 0
    for j in range(L):
        r0, r1 = O.grid_res(d, j)
        assert O.grid_offset(d, j, 0) == off
        off += r0 * r0 * d.c0
        assert O.grid_offset(d, j, 1) == off
        off += r1 * r1 * d.c1
    assert O.num_latents(d) == off
    # 4096^2 NTC 0.2 has 12,303,280 latents
    assert O.num_latents(Profile.named("ntc0.2", 4096, 9)) == 12_303_280
    assert O.num_latents(Profile.named("ntc0.2", 2048, 9)) == 3_075_820


@pytest.mark.parametrize("name", ["ntc0.2", "ntc1.0"])
@pytest.mark.parametrize("W", [16, 32, 64])
def test_taps_brute_force_integer(O, name, W):
    """Every (m, x, y) of small chains: tap indices equal an integer re-derivation
    floor(((2x+1) r - w_m) / (2 w_m)) (+0/+1, clamped), bilinear weights sum to 1 and
    are the fractional offsets ((2x+1) r - w_m) mod 2w_m / 2w_m."""
    d = Profile.named(name, W, 4)
    M = O.num_mips(W)
    for m in range(M):
        wm = W >> m
        j = O.level_of_mip(d, m)
        r = O.grid_res(d, j)
        for y in range(wm):
            for x in range(wm):
                ti, tw = O.address(d, m, x, y)
                assert ti[0] == j
                for k in range(2):
                    num_x, num_y = (2 * x + 1) * r[k] - wm, (2 * y + 1) * r[k] - wm
                    ix, iy = num_x // (2 * wm), num_y // (2 * wm)
                    for t in range(4):
                        ex = min(max(ix + (t & 1), 0), r[k] - 1)
                        ey = min(max(iy + (t >> 1), 0), r[k] - 1)
                        assert (ti[1 + 8 * k + 2 * t], ti[2 + 8 * k + 2 * t]) == (ex, ey)
                    if k == 1:
                        fx = (num_x % (2 * wm)) / (2 * wm)
                        fy = (num_y % (2 * wm)) / (2 * wm)
                        want = [(1 - fx) * (1 - fy), fx * (1 - fy), (1 - fx) * fy, fx * fy]
                        assert np.allclose(tw, want, atol=0, rtol=0) or np.allclose(tw, want, atol=1e-15)
                        assert abs(tw.sum() - 1.0) < 1e-15


def test_addressing_closed_forms(O):
    """SPEC.md:171, 180-182 and north_star: a 1:1 grid reproduces the cell at texel
    centres; a 1x1 grid gives four identical taps; a 2x downsample takes the 2x2 footprint."""
    d = Profile.named("ntc0.2", 64, 4)  # G0 16, G1 8 at level 0
    # mip 2: w_m = 16 = r0 -> G0 1:1; mip 3: w_m = 8 = r1 -> G1 1:1
    for x in range(16):
        ti, _ = O.address(d, 2, x, 5)
        assert (ti[1], ti[2]) == (x, 5)
    for x in range(8):
        ti, tw = O.address(d, 3, x, 3)
        assert (ti[9], ti[10]) == (x, 3)
        assert tw[0] == 1.0 and tw[1] == tw[2] == tw[3] == 0.0
    # mip 3 for G0 (r0 = 16, w_m = 8): 2x downsample -> taps 2x, 2x+1, weights irrelevant
    for x in range(8):
        ti, _ = O.address(d, 3, x, x)
        assert [ti[1], ti[3]] == [2 * x, 2 * x + 1]
        assert [ti[2], ti[6]] == [2 * x, 2 * x + 1]
    # the last level's G1 is 1x1 at 128^2 (32 -> 8 -> 2) -> four identical taps
    d = Profile.named("ntc0.2", 128, 4)
    L = O.num_levels(d)
    assert O.grid_res(d, L - 1) == (2, 1)
    ti, tw = O.address(d, O.num_mips(128) - 1, 0, 0)
    assert set(ti[9:17].tolist()) == {0}


def test_g1_bilinear_matches_grid_sample(O):
    """The G1 part of the assembled input equals torch grid_sample (bilinear,
    align_corners=False, border padding: texel-centre mapping with edge clamp) of the
    dequantised grid, rounded to fp16 -- an independent library implementation."""
    d = Profile.named("ntc0.2", 64, 4)
    L = O.num_levels(d)
    grids = []
    for j in range(L):
        r0, r1 = O.grid_res(d, j)
        grids += [(r0 * r0 * d.c0, d.b0), (r1 * r1 * d.c1, d.b1)]
    codes = gen_codes(7, grids)
    for m in range(O.num_mips(64)):
        j = O.level_of_mip(d, m)
        r0, r1 = O.grid_res(d, j)
        off = O.grid_offset(d, j, 1)
        g = codes[off: off + r1 * r1 * d.c1].reshape(r1, r1, d.c1).astype(np.float64)
        g = (g - (2 ** d.b1 // 2 - 1)) / 2 ** d.b1
        wm = 64 >> m
        ys, xs = np.meshgrid(np.arange(wm), np.arange(wm), indexing="ij")
        gx = (xs + 0.5) / wm * 2 - 1
        gy = (ys + 0.5) / wm * 2 - 1
        grid = torch.tensor(np.stack([gx, gy], -1)[None], dtype=torch.float64)
        inp = torch.tensor(g.transpose(2, 0, 1)[None], dtype=torch.float64)
        ref = torch.nn.functional.grid_sample(inp, grid, mode="bilinear", padding_mode="border",
                                              align_corners=False)[0].numpy().transpose(1, 2, 0)
        ref16 = ref.astype(np.float16)
        for y in range(0, wm, max(1, wm // 8)):
            for x in range(wm):
                X = O.assemble(d, codes, m, x, y).view(np.float16)
                got = X[4 * d.c0: 4 * d.c0 + d.c1]
                assert np.array_equal(got, ref16[y, x]), (m, x, y)


def test_g0_taps_match_unfiltered_cells(O):
    """G0 part of X = the 4 dequantised cells at the taps (tap-major, channel-minor)."""
    d = Profile.named("ntc0.2", 32, 4)
    L = O.num_levels(d)
    grids = []
    for j in range(L):
        r0, r1 = O.grid_res(d, j)
        grids += [(r0 * r0 * d.c0, d.b0), (r1 * r1 * d.c1, d.b1)]
    codes = gen_codes(3, grids)
    for m in range(O.num_mips(32)):
        wm = 32 >> m
        j = O.level_of_mip(d, m)
        r0, _ = O.grid_res(d, j)
        off = O.grid_offset(d, j, 0)
        g = codes[off: off + r0 * r0 * d.c0].reshape(r0, r0, d.c0)
        for y in range(wm):
            for x in range(wm):
                ti, _ = O.address(d, m, x, y)
                X = O.assemble(d, codes, m, x, y).view(np.float16).astype(np.float64)
                for t in range(4):
                    cell = g[ti[2 + 2 * t], ti[1 + 2 * t]]
                    want = (cell.astype(np.float64) - 1) / 4
                    assert np.array_equal(X[t * 8:(t + 1) * 8], want)
