"""CPU ORACLE FOR TESTS ONLY -- test infrastructure, not product code.

ctypes marshalling around ``oracle/libntc_oracle.so`` (plain scalar fp64 C, see
``ntc_oracle.c``).  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this module.  The CUDA product
path (``paper_2305_17105_b200``) never imports it and shares no code with it.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libntc_oracle.so")
_SRC = os.path.join(_HERE, "ntc_oracle.c")


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (-O2, no fast-math, OpenMP)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
        os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "ntc_oracle.h"))
    ):
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-fopenmp", "-fPIC", "-shared", "-o", _SO, _SRC, "-lm"]
        )
    return _SO


class Desc(ctypes.Structure):
    _fields_ = [
        ("width", ctypes.c_int32),
        ("channels", ctypes.c_int32),
        ("g0_ratio", ctypes.c_int32),
        ("c0", ctypes.c_int32),
        ("b0", ctypes.c_int32),
        ("c1", ctypes.c_int32),
        ("b1", ctypes.c_int32),
        ("hidden_mats", ctypes.c_int32),
        ("activation", ctypes.c_int32),
    ]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        L = _lib
        P = ctypes.POINTER
        i32, i64, f64, u16, u64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_uint16, ctypes.c_uint64
        vp = ctypes.c_void_p
        sig = {
            "ntco_num_mips": (i32, [i32]),
            "ntco_num_levels": (i32, [P(Desc)]),
            "ntco_level_of_mip": (i32, [P(Desc), i32]),
            "ntco_grid_res": (None, [P(Desc), i32, P(i32), P(i32)]),
            "ntco_grid_offset": (i64, [P(Desc), i32, i32]),
            "ntco_num_latents": (i64, [P(Desc)]),
            "ntco_input_dim": (i32, [P(Desc)]),
            "ntco_num_params": (i64, [P(Desc)]),
            "ntco_address": (None, [P(Desc), i32, i32, i32, vp, vp]),
            "ntco_quantize": (i32, [f64, i32]),
            "ntco_dequantize": (f64, [i32, i32]),
            "ntco_quant_lo": (f64, [i32]),
            "ntco_quant_hi": (f64, [i32]),
            "ntco_quantize_latents": (None, [P(Desc), vp, vp]),
            "ntco_tri": (f64, [f64]),
            "ntco_pe": (None, [i32, i32, vp]),
            "ntco_f64_to_f16": (u16, [f64]),
            "ntco_f16_to_f64": (f64, [u16]),
            "ntco_lod_f16": (u16, [i32, i32]),
            "ntco_assemble": (None, [P(Desc), vp, i32, i32, i32, vp]),
            "ntco_hardgelu": (f64, [f64]),
            "ntco_hardgelu_grad": (f64, [f64]),
            "ntco_gelu": (f64, [f64]),
            "ntco_gelu_grad": (f64, [f64]),
            "ntco_mlp_forward": (None, [P(Desc), vp, vp, vp]),
            "ntco_decode_texels": (None, [P(Desc), vp, vp, vp, i64, vp, i32]),
            "ntco_decode_mip": (None, [P(Desc), vp, vp, i32, vp, i32]),
            "ntco_philox4x32_10": (None, [vp, vp, vp]),
            "ntco_filter": (None, [P(Desc), vp, vp, vp, i64, i32, u64, vp, i32]),
            "ntco_noise": (f64, [u64, ctypes.c_uint32, i64, i32]),
            "ntco_train_grads": (
                f64,
                [P(Desc), vp, vp, i32, i32, vp, vp, u64, ctypes.c_uint32, i32, i32, vp, vp, i32],
            ),
            "ntco_adam": (
                None,
                [i64, vp, vp, vp, vp, i32, f64, f64, f64, f64, i32, i32, f64, f64],
            ),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
    return _lib


def _p(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.c_void_p)


def desc(width, channels, g0_ratio=4, c0=8, b0=2, c1=12, b1=4, hidden_mats=1, activation=0) -> Desc:
    return Desc(width, channels, g0_ratio, c0, b0, c1, b1, hidden_mats, activation)


def desc_from(d) -> Desc:
    """Accept a Desc or any object with the same attribute names (e.g. synth.Profile)."""
    if isinstance(d, Desc):
        return d
    return Desc(*[int(getattr(d, f)) for f, _ in Desc._fields_])


# ---- thin wrappers -------------------------------------------------------------------
def num_mips(width):
    return lib().ntco_num_mips(width)


def num_levels(d):
    return lib().ntco_num_levels(ctypes.byref(desc_from(d)))


def level_of_mip(d, m):
    return lib().ntco_level_of_mip(ctypes.byref(desc_from(d)), m)


def grid_res(d, j):
    r0, r1 = ctypes.c_int32(), ctypes.c_int32()
    lib().ntco_grid_res(ctypes.byref(desc_from(d)), j, ctypes.byref(r0), ctypes.byref(r1))
    return r0.value, r1.value


def grid_offset(d, j, k):
    return lib().ntco_grid_offset(ctypes.byref(desc_from(d)), j, k)


def num_latents(d):
    return lib().ntco_num_latents(ctypes.byref(desc_from(d)))


def input_dim(d):
    return lib().ntco_input_dim(ctypes.byref(desc_from(d)))


def num_params(d):
    return lib().ntco_num_params(ctypes.byref(desc_from(d)))


def address(d, m, x, y):
    oi = np.zeros(17, np.int32)
    ow = np.zeros(4, np.float64)
    lib().ntco_address(ctypes.byref(desc_from(d)), m, x, y, _p(oi), _p(ow))
    return oi, ow


def quantize(v, bits):
    return lib().ntco_quantize(float(v), bits)


def dequantize(code, bits):
    return lib().ntco_dequantize(int(code), bits)


def quant_range(bits):
    return lib().ntco_quant_lo(bits), lib().ntco_quant_hi(bits)


def quantize_latents(d, latents: np.ndarray) -> np.ndarray:
    lat = np.ascontiguousarray(latents, np.float32)
    out = np.zeros(lat.shape, np.uint8)
    lib().ntco_quantize_latents(ctypes.byref(desc_from(d)), _p(lat), _p(out))
    return out


def tri(t):
    return lib().ntco_tri(float(t))


def pe(x, y):
    out = np.zeros(12, np.float64)
    lib().ntco_pe(x, y, _p(out))
    return out


def f64_to_f16(v):
    return lib().ntco_f64_to_f16(float(v))


def f16_to_f64(h):
    return lib().ntco_f16_to_f64(int(h))


def lod_f16(m, M):
    return lib().ntco_lod_f16(m, M)


def assemble(d, codes, m, x, y) -> np.ndarray:
    dd = desc_from(d)
    X = np.zeros(lib().ntco_input_dim(ctypes.byref(dd)), np.uint16)
    codes = np.ascontiguousarray(codes, np.uint8)
    lib().ntco_assemble(ctypes.byref(dd), _p(codes), m, x, y, _p(X))
    return X


def hardgelu(x):
    return lib().ntco_hardgelu(float(x))


def hardgelu_grad(x):
    return lib().ntco_hardgelu_grad(float(x))


def gelu(x):
    return lib().ntco_gelu(float(x))


def gelu_grad(x):
    return lib().ntco_gelu_grad(float(x))


def mlp_forward(d, params: np.ndarray, X: np.ndarray) -> np.ndarray:
    dd = desc_from(d)
    params = np.ascontiguousarray(params, np.float64)
    X = np.ascontiguousarray(X, np.float64)
    y = np.zeros(dd.channels, np.float64)
    lib().ntco_mlp_forward(ctypes.byref(dd), _p(params), _p(X), _p(y))
    return y


def decode_texels(d, codes, weights_f16, queries_xym: np.ndarray, nthreads: int = 0) -> np.ndarray:
    """queries_xym: (n, 3) int32 (x, y, mip).  Returns (n, c) float64."""
    dd = desc_from(d)
    q = np.ascontiguousarray(queries_xym, np.int32)
    codes = np.ascontiguousarray(codes, np.uint8)
    w = np.ascontiguousarray(weights_f16, np.uint16)
    out = np.zeros((q.shape[0], dd.channels), np.float64)
    lib().ntco_decode_texels(ctypes.byref(dd), _p(codes), _p(w), _p(q), q.shape[0], _p(out), nthreads)
    return out


def decode_mip(d, codes, weights_f16, m, nthreads: int = 0) -> np.ndarray:
    dd = desc_from(d)
    wm = dd.width >> m
    codes = np.ascontiguousarray(codes, np.uint8)
    w = np.ascontiguousarray(weights_f16, np.uint16)
    out = np.zeros((wm, wm, dd.channels), np.float64)
    lib().ntco_decode_mip(ctypes.byref(dd), _p(codes), _p(w), m, _p(out), nthreads)
    return out


def filter_texels(d, codes, weights_f16, uvl, mode, seed=0, nthreads=0) -> np.ndarray:
    """uvl: (n, 3) float64 (u, v, lod); mode 0 nearest, 1 bilinear, 2 trilinear, 3 stochastic
    bilinear, 4 stochastic trilinear.  Returns (n, c) float64."""
    dd = desc_from(d)
    q = np.ascontiguousarray(uvl, np.float64)
    codes = np.ascontiguousarray(codes, np.uint8)
    w = np.ascontiguousarray(weights_f16, np.uint16)
    out = np.zeros((q.shape[0], dd.channels), np.float64)
    lib().ntco_filter(ctypes.byref(dd), _p(codes), _p(w), _p(q), q.shape[0], mode, seed, _p(out), nthreads)
    return out


def philox(ctr, key) -> np.ndarray:
    c = np.ascontiguousarray(ctr, np.uint32)
    k = np.ascontiguousarray(key, np.uint32)
    o = np.zeros(4, np.uint32)
    lib().ntco_philox4x32_10(_p(c), _p(k), _p(o))
    return o


def noise(seed, step, idx, bits):
    return lib().ntco_noise(seed, step, idx, bits)


def train_grads(d, latents, params_f32, mip, crops, ref_f16, seed, step, noise_on=True, nthreads=0,
                round_f16=True):
    """Returns (loss, dparams[P] float64, dlatents[NL] float64)."""
    dd = desc_from(d)
    lat = np.ascontiguousarray(latents, np.float32)
    par = np.ascontiguousarray(params_f32, np.float32)
    cr = np.ascontiguousarray(crops, np.int32).reshape(-1, 4)
    ref = np.ascontiguousarray(ref_f16, np.uint16)
    dp = np.zeros(num_params(dd), np.float64)
    dl = np.zeros(num_latents(dd), np.float64)
    loss = lib().ntco_train_grads(
        ctypes.byref(dd), _p(lat), _p(par), mip, cr.shape[0], _p(cr), _p(ref),
        seed, step, int(noise_on), int(round_f16), _p(dp), _p(dl), nthreads,
    )
    return loss, dp, dl


def adam(p, m, v, g, t, lr, beta1=0.9, beta2=0.999, eps=1e-8, sparse=False, clamp=None):
    """In-place Adam on float32 arrays; clamp=(lo, hi) or None."""
    for a in (p, m, v, g):
        assert a.dtype == np.float32 and a.flags["C_CONTIGUOUS"]
    lo, hi = clamp if clamp is not None else (0.0, 0.0)
    lib().ntco_adam(p.size, _p(p), _p(m), _p(v), _p(g), t, lr, beta1, beta2, eps,
                    int(sparse), int(clamp is not None), lo, hi)
