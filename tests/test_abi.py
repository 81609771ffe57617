"""CPU checks of the C-ABI library: it builds, loads, exports every symbol include/ntc.h
declares, and its host-side geometry / argument validation match the oracle (no GPU)."""
import ctypes
import os
import re
import subprocess

import pytest

import paper_2305_17105_b200 as ntc
from paper_2305_17105_b200 import build as ntc_build
from paper_2305_17105_b200.synth import Profile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def libpath():
    return ntc_build.build()


def _declared():
    src = open(os.path.join(ROOT, "include", "ntc.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ntc_[a-z_0-9]+)\s*\(", src)))


def test_exports_every_declared_symbol(libpath):
    names = _declared()
    assert "ntc_decode_texels" in names and "ntc_decode_mip" in names and "ntc_train_step" in names
    out = subprocess.check_output(["nm", "-D", "--defined-only", libpath], text=True)
    exported = set(re.findall(r"\bT (ntc_[a-z_0-9]+)\b", out))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    for n in names:
        assert n in ntc.ABI_FUNCTIONS, n
        getattr(ntc.lib(), n)


def test_sm100a_code_only(libpath):
    out = subprocess.check_output(["cuobjdump", "--list-elf", libpath], text=True)
    assert "sm_100a" in out
    sass = subprocess.check_output(["cuobjdump", "-sass", libpath], text=True)
    assert "UTCHMMA" in sass  # tcgen05.mma
    assert "LDTM" in sass      # tcgen05.ld
    assert " HMMA" not in sass  # no legacy mma.sync path


@pytest.mark.parametrize("name", ["ntc0.2", "ntc0.5", "ntc1.0", "ntc2.25"])
def test_host_geometry_matches_oracle(O, libpath, name):
    for W in (8, 16, 256, 1024, 2048, 4096, 8192):
        d = Profile.named(name, W, 9)
        if W // d.g0_ratio < 2:
            continue
        assert ntc.ntc_num_mips(d) == O.num_mips(W)
        assert ntc.ntc_num_levels(d) == O.num_levels(d)
        assert ntc.ntc_num_latents(d) == O.num_latents(d)
        assert ntc.ntc_num_params(d) == O.num_params(d)
        for m in range(O.num_mips(W)):
            assert ntc.ntc_level_of_mip(d, m) == O.level_of_mip(d, m)
        for j in range(O.num_levels(d)):
            r0, r1, o0, o1 = ntc.ntc_grid_layout(d, j)
            assert (r0, r1) == O.grid_res(d, j)
            assert (o0, o1) == (O.grid_offset(d, j, 0), O.grid_offset(d, j, 1))
        assert ntc.ntc_chain_texels(d) == sum((W >> m) ** 2 for m in range(O.num_mips(W)))


def test_host_validation_without_gpu(libpath):
    L = ntc.lib()
    bad_profile = ntc.make_desc(Profile(64, 8, 4, 6, 3, 12, 4))
    assert L.ntc_quantize_latents(ctypes.byref(bad_profile), None, None, None) == ntc.NTC_ERR_UNSUPPORTED
    for bad, msg in ((Profile(63, 8), b"width"), (Profile(64, 0), b"channels"), (Profile(64, 17), b"channels"),
                     (Profile(64, 8, 3), b"g0_ratio"), (Profile(64, 8, 0), b"g0_ratio"),
                     (Profile(64, 8, hidden_mats=3), b"hidden_mats")):
        assert L.ntc_quantize_latents(ctypes.byref(ntc.make_desc(bad)), None, None, None) == \
            ntc.NTC_ERR_INVALID_ARGUMENT
        assert msg in L.ntc_last_error(), (bad, L.ntc_last_error())
        # the trainer validates the same descriptor before touching the device
        out = ctypes.c_void_p()
        assert L.ntc_trainer_create(ctypes.byref(ntc.make_desc(bad)), ctypes.byref(out)) == \
            ntc.NTC_ERR_INVALID_ARGUMENT
        assert msg in L.ntc_last_error(), (bad, L.ntc_last_error())
    ok = ntc.make_desc(Profile.named("ntc0.2", 64, 8))
    assert L.ntc_quantize_latents(ctypes.byref(ok), None, None, None) == ntc.NTC_ERR_INVALID_ARGUMENT
    assert L.ntc_decode_chain(None, None, None) == ntc.NTC_ERR_INVALID_ARGUMENT
    assert L.ntc_decode_texels(None, None, 0, None, None, None) == ntc.NTC_ERR_INVALID_ARGUMENT


def test_product_has_no_oracle_dependency():
    """The product package never imports / links the oracle (parity rules)."""
    pkg = os.path.join(ROOT, "paper_2305_17105_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "ntc_oracle" not in txt and "ntco_" not in txt, f


@pytest.mark.parametrize("mip", [0, 1, 3, 5])
def test_train_footprint_matches_oracle(O, libpath, mip):
    """Host footprint boxes (disjoint) cover exactly the latent cells the batch reads
    according to the oracle's addressing."""
    import numpy as np

    from paper_2305_17105_b200.synth import gen_crops

    d = Profile.named("ntc0.2", 128, 8)
    crops = gen_crops(3 + mip, 128, mip, 5, 24 >> min(mip, 2))
    b = ntc.make_batch(mip, crops, None, 0)
    boxes = ntc.ntc_train_footprint(d, b)
    got = set()
    for lvl, k, x0, y0, x1, y1 in boxes:
        for y in range(y0, y1 + 1):
            for x in range(x0, x1 + 1):
                cell = (lvl, k, x, y)
                assert cell not in got  # disjoint
                got.add(cell)
    want = set()
    for x0, y0, w, h in crops:
        for y in range(y0, y0 + h):
            for x in range(x0, x0 + w):
                ti, _ = O.address(d, mip, x, y)
                for t in range(4):
                    want.add((ti[0], 0, ti[1 + 2 * t], ti[2 + 2 * t]))
                    want.add((ti[0], 1, ti[9 + 2 * t], ti[10 + 2 * t]))
    assert got == want


def test_missing_library_fails_loudly(monkeypatch):
    """No CPU fallback: with the CUDA library absent every call raises instead of computing."""
    import paper_2305_17105_b200 as ntc

    monkeypatch.setattr(ntc, "_lib", None)
    monkeypatch.setattr(ntc, "LIB_PATH", "/nonexistent/libntc.so")
    with pytest.raises(RuntimeError, match="library missing"):
        ntc.lib()
    with pytest.raises(RuntimeError, match="library missing"):
        ntc.ntc_chain_texels(Profile.named("ntc0.2", 64, 8))
