"""Python binding of the NTC B200 C ABI (include/ntc.h) -- argument marshalling only.

Every step of the hot path runs in the CUDA library ``libntc.so`` built in-tree for
sm_100a (``python -m paper_2305_17105_b200.build`` or ``__graft_entry__.build()``).
There is no CPU fallback: if the library is missing, every call raises.  PyTorch is used
for device memory and streams only; tensors are passed to the ABI as raw pointers.
"""
from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libntc.so")

NTC_OK = 0
NTC_ERR_INVALID_ARGUMENT = 1
NTC_ERR_OUT_OF_RANGE = 2
NTC_ERR_DATA = 3
NTC_ERR_NONFINITE = 4
NTC_ERR_CUDA = 5
NTC_ERR_UNSUPPORTED = 6
NTC_STEP_GRADS = 1
NTC_STEP_APPLY = 2
NTC_MAX_CROPS = 64


class NtcError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"ntc status {status}: {msg}")
        self.status = status


class Desc(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in
                ("width", "channels", "g0_ratio", "c0", "b0", "c1", "b1", "hidden_mats", "activation")]


class TrainBuffers(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in
                ("latents", "m_lat", "v_lat", "grad_lat", "params", "m_par", "v_par", "grad_par", "noisy")]


class Batch(ctypes.Structure):
    _fields_ = [("mip", ctypes.c_int32), ("n_crops", ctypes.c_int32), ("crops", ctypes.c_void_p),
                ("ref", ctypes.c_void_p), ("ref_row_stride_elems", ctypes.c_int64), ("norm_texels", ctypes.c_int64)]


class Hparams(ctypes.Structure):
    _fields_ = [("lr_latent", ctypes.c_float), ("lr_weight", ctypes.c_float), ("beta1", ctypes.c_float),
                ("beta2", ctypes.c_float), ("eps", ctypes.c_float), ("step", ctypes.c_int32),
                ("seed", ctypes.c_uint64), ("noise_on", ctypes.c_int32), ("dense_latent_adam", ctypes.c_int32),
                ("freeze_latents", ctypes.c_int32)]


ABI_FUNCTIONS = {
    # name: (restype, argtypes)
    "ntc_last_error": (ctypes.c_char_p, []),
    "ntc_num_mips": (ctypes.c_int32, [ctypes.c_void_p]),
    "ntc_num_levels": (ctypes.c_int32, [ctypes.c_void_p]),
    "ntc_level_of_mip": (ctypes.c_int32, [ctypes.c_void_p, ctypes.c_int32]),
    "ntc_grid_layout": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32] + [ctypes.c_void_p] * 4),
    "ntc_num_latents": (ctypes.c_int64, [ctypes.c_void_p]),
    "ntc_num_params": (ctypes.c_int64, [ctypes.c_void_p]),
    "ntc_chain_texels": (ctypes.c_int64, [ctypes.c_void_p]),
    "ntc_mip_offset": (ctypes.c_int64, [ctypes.c_void_p, ctypes.c_int32]),
    "ntc_quantize_latents": (ctypes.c_int, [ctypes.c_void_p] * 4),
    "ntc_dequantize_codes": (ctypes.c_int, [ctypes.c_void_p] * 4),
    "ntc_material_create": (ctypes.c_int, [ctypes.c_void_p] * 5),
    "ntc_material_destroy": (None, [ctypes.c_void_p]),
    "ntc_decode_texels": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                         ctypes.c_void_p, ctypes.c_void_p]),
    "ntc_decode_mip": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_int64,
                                      ctypes.c_void_p]),
    "ntc_decode_chain": (ctypes.c_int, [ctypes.c_void_p] * 3),
    "ntc_decode_chain_part": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p,
                                             ctypes.c_void_p]),
    "ntc_decode_multi_scratch_bytes": (ctypes.c_int64, [ctypes.c_int64]),
    "ntc_decode_texels_multi": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_int64,
                                               ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                               ctypes.c_void_p]),
    "ntc_footprint_size": (ctypes.c_int64, [ctypes.c_void_p] * 2),
    "ntc_boxes_size": (ctypes.c_int64, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32]),
    "ntc_boxes_copy": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p,
                                      ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p]),
    "ntc_train_apply_boxes": (ctypes.c_int, [ctypes.c_void_p] * 4 + [ctypes.c_int32, ctypes.c_void_p,
                                                                     ctypes.c_void_p]),
    "ntc_filter_scratch_bytes": (ctypes.c_int64, [ctypes.c_int64, ctypes.c_int32, ctypes.c_int32]),
    "ntc_filter_texels": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32,
                                         ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "ntc_footprint_pack": (ctypes.c_int, [ctypes.c_void_p] * 5),
    "ntc_footprint_unpack": (ctypes.c_int, [ctypes.c_void_p] * 5),
    "ntc_debug_assemble": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                          ctypes.c_void_p, ctypes.c_void_p]),
    "ntc_trainer_create": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p]),
    "ntc_trainer_destroy": (None, [ctypes.c_void_p]),
    "ntc_train_step": (ctypes.c_int, [ctypes.c_void_p] * 7 + [ctypes.c_uint32, ctypes.c_void_p]),
    "ntc_train_footprint": (ctypes.c_int32, [ctypes.c_void_p] * 3),
}

_lib = None


def lib() -> ctypes.CDLL:
    """Load the in-tree CUDA library; raise loudly if it was not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"NTC CUDA library missing: {LIB_PATH} (run __graft_entry__.build())")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in ABI_FUNCTIONS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _check(status: int):
    if status != NTC_OK:
        raise NtcError(status, lib().ntc_last_error().decode())


def _ptr(t):
    if t is None:
        return None
    if isinstance(t, torch.Tensor):
        return ctypes.c_void_p(t.data_ptr())
    return t


def _stream(stream=None):
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


_DESC_CACHE = {}


def make_desc(p) -> Desc:
    """From any object with the ntc_desc field names (e.g. synth.Profile); cached per value
    (the hot-path wrappers are called every training step)."""
    if isinstance(p, Desc):
        return p
    key = tuple(int(getattr(p, f)) for f, _ in Desc._fields_)
    d = _DESC_CACHE.get(key)
    if d is None:
        d = _DESC_CACHE[key] = Desc(*key)
    return d


# ---------------------------------------------------------------- geometry (host)
def ntc_num_mips(d):
    return lib().ntc_num_mips(ctypes.byref(make_desc(d)))


def ntc_num_levels(d):
    return lib().ntc_num_levels(ctypes.byref(make_desc(d)))


def ntc_level_of_mip(d, mip):
    return lib().ntc_level_of_mip(ctypes.byref(make_desc(d)), mip)


def ntc_grid_layout(d, level):
    r0, r1 = ctypes.c_int32(), ctypes.c_int32()
    o0, o1 = ctypes.c_int64(), ctypes.c_int64()
    _check(lib().ntc_grid_layout(ctypes.byref(make_desc(d)), level, ctypes.byref(r0), ctypes.byref(r1),
                                 ctypes.byref(o0), ctypes.byref(o1)))
    return r0.value, r1.value, o0.value, o1.value


def ntc_num_latents(d):
    return lib().ntc_num_latents(ctypes.byref(make_desc(d)))


def ntc_num_params(d):
    return lib().ntc_num_params(ctypes.byref(make_desc(d)))


def ntc_chain_texels(d):
    return lib().ntc_chain_texels(ctypes.byref(make_desc(d)))


def ntc_mip_offset(d, mip):
    return lib().ntc_mip_offset(ctypes.byref(make_desc(d)), mip)


def grid_list(d):
    """[(n_values, bits)] per grid in canonical order (for synth.gen_codes)."""
    out = []
    for j in range(ntc_num_levels(d)):
        r0, r1, _, _ = ntc_grid_layout(d, j)
        out += [(r0 * r0 * d.c0, d.b0), (r1 * r1 * d.c1, d.b1)]
    return out


# ---------------------------------------------------------------- a0
def ntc_quantize_latents(d, latents: torch.Tensor, codes: torch.Tensor, stream=None):
    assert latents.is_cuda and latents.dtype == torch.float32 and codes.dtype == torch.uint8
    _check(lib().ntc_quantize_latents(ctypes.byref(make_desc(d)), _ptr(latents), _ptr(codes), _stream(stream)))


def ntc_dequantize_codes(d, codes: torch.Tensor, latents: torch.Tensor, stream=None):
    assert codes.dtype == torch.uint8 and latents.dtype == torch.float32
    _check(lib().ntc_dequantize_codes(ctypes.byref(make_desc(d)), _ptr(codes), _ptr(latents), _stream(stream)))


# ---------------------------------------------------------------- material + decode
class Material:
    """Device-resident material (packed grids + swizzled weights), owned by the library."""

    def __init__(self, d, codes: torch.Tensor, weights_f16: torch.Tensor, stream=None):
        assert codes.is_cuda and codes.dtype == torch.uint8 and codes.is_contiguous()
        assert weights_f16.is_cuda and weights_f16.element_size() == 2 and weights_f16.is_contiguous()
        self.profile = d
        self.desc = make_desc(d)
        h = ctypes.c_void_p()
        _check(lib().ntc_material_create(ctypes.byref(self.desc), _ptr(codes), _ptr(weights_f16),
                                         _stream(stream), ctypes.byref(h)))
        self.handle = h

    def close(self):
        if getattr(self, "handle", None):
            lib().ntc_material_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def pack_queries(xym: torch.Tensor, material: torch.Tensor = None) -> torch.Tensor:
    """(n, 3) int tensor (x, y, mip) [+ material index per query] -> int64 [n] holding
    ntc_query structs (8 bytes)."""
    x, y, m = xym[:, 0].long(), xym[:, 1].long(), xym[:, 2].long()
    q = (x & 0xFFFF) | ((y & 0xFFFF) << 16) | ((m & 0xFF) << 32)
    if material is not None:
        q = q | ((material.long().to(q.device) & 0xFF) << 40)
    return q


def ntc_decode_texels(mat: Material, queries: torch.Tensor, out: torch.Tensor, status: torch.Tensor = None,
                      stream=None):
    assert queries.dtype == torch.int64 and out.dtype == torch.float16
    _check(lib().ntc_decode_texels(mat.handle, _ptr(queries), queries.numel(), _ptr(out), _ptr(status),
                                   _stream(stream)))


def ntc_decode_multi_scratch_bytes(n: int) -> int:
    return int(lib().ntc_decode_multi_scratch_bytes(n))


def ntc_decode_texels_multi(mats, queries: torch.Tensor, out: torch.Tensor, status: torch.Tensor = None,
                            scratch: torch.Tensor = None, stream=None):
    """Queries of several materials (index in bits 40-47, see pack_queries) in one call."""
    assert queries.dtype == torch.int64 and out.dtype == torch.float16
    n = queries.numel()
    need = ntc_decode_multi_scratch_bytes(n)
    if scratch is None:
        scratch = torch.empty(need, dtype=torch.uint8, device=queries.device)
    arr = (ctypes.c_void_p * len(mats))(*[m.handle.value for m in mats])
    _check(lib().ntc_decode_texels_multi(arr, len(mats), _ptr(queries), n, _ptr(out), _ptr(status), _ptr(scratch),
                                         scratch.numel() * scratch.element_size(), _stream(stream)))
    return scratch


def ntc_decode_mip(mat: Material, mip: int, out: torch.Tensor, row_stride_elems: int = None, stream=None):
    assert out.dtype == torch.float16
    if row_stride_elems is None:
        row_stride_elems = (mat.desc.width >> mip) * mat.desc.channels
    _check(lib().ntc_decode_mip(mat.handle, mip, _ptr(out), row_stride_elems, _stream(stream)))


def ntc_decode_chain(mat: Material, out: torch.Tensor, stream=None):
    assert out.dtype == torch.float16 and out.numel() >= ntc_chain_texels(mat.profile) * mat.desc.channels
    _check(lib().ntc_decode_chain(mat.handle, _ptr(out), _stream(stream)))


NTC_FILTER_NEAREST, NTC_FILTER_BILINEAR, NTC_FILTER_TRILINEAR = 0, 1, 2
NTC_FILTER_STOCHASTIC_BILINEAR, NTC_FILTER_STOCHASTIC_TRILINEAR = 3, 4


def ntc_filter_texels(mat: Material, uvl: torch.Tensor, mode: int, out: torch.Tensor, seed: int = 0,
                      scratch: torch.Tensor = None, stream=None):
    """uvl: device fp32 (n, 3) = (u, v, lod); out: device fp16 (n, c)."""
    assert uvl.dtype == torch.float32 and out.dtype == torch.float16
    n = uvl.shape[0]
    if scratch is None:
        nb = lib().ntc_filter_scratch_bytes(n, mode, mat.desc.channels)
        scratch = torch.empty(max(nb, 256), dtype=torch.uint8, device=uvl.device)
    _check(lib().ntc_filter_texels(mat.handle, _ptr(uvl), n, mode, seed, _ptr(out), _ptr(scratch), _stream(stream)))


def ntc_decode_chain_part(mat: Material, part: int, nparts: int, out: torch.Tensor, stream=None):
    assert out.dtype == torch.float16 and out.numel() >= ntc_chain_texels(mat.profile) * mat.desc.channels
    _check(lib().ntc_decode_chain_part(mat.handle, part, nparts, _ptr(out), _stream(stream)))


def ntc_debug_assemble(mat: Material, queries: torch.Tensor, addr: torch.Tensor, X: torch.Tensor, stream=None):
    _check(lib().ntc_debug_assemble(mat.handle, _ptr(queries), queries.numel(), _ptr(addr), _ptr(X),
                                    _stream(stream)))


# ---------------------------------------------------------------- training
class Trainer:
    def __init__(self, d):
        self.profile = d
        self.desc = make_desc(d)
        h = ctypes.c_void_p()
        _check(lib().ntc_trainer_create(ctypes.byref(self.desc), ctypes.byref(h)))
        self.handle = h

    def close(self):
        if getattr(self, "handle", None):
            lib().ntc_trainer_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def make_batch(mip: int, crops, ref: torch.Tensor, ref_row_stride_elems: int, norm_texels: int = 0):
    """crops: host int32 contiguous (n, 4) array-like (kept alive by the returned tuple)."""
    import numpy as np

    cr = np.ascontiguousarray(np.asarray(crops, dtype=np.int32).reshape(-1, 4))
    b = Batch(mip, cr.shape[0], cr.ctypes.data_as(ctypes.c_void_p), _ptr(ref), ref_row_stride_elems, norm_texels)
    return b, cr


def make_buffers(t: dict) -> TrainBuffers:
    return TrainBuffers(*[_ptr(t[n]) for n, _ in TrainBuffers._fields_])


def ntc_train_step(trainer: Trainer, buffers: TrainBuffers, batch, hp: Hparams, loss: torch.Tensor,
                   status: torch.Tensor = None, flags: int = NTC_STEP_GRADS | NTC_STEP_APPLY, stream=None):
    b = batch[0] if isinstance(batch, tuple) else batch
    _check(lib().ntc_train_step(trainer.handle, ctypes.byref(trainer.desc), ctypes.byref(buffers), ctypes.byref(b),
                                ctypes.byref(hp), _ptr(loss), _ptr(status), flags, _stream(stream)))


def ntc_train_footprint(d, batch):
    import numpy as np

    b = batch[0] if isinstance(batch, tuple) else batch
    n = lib().ntc_train_footprint(ctypes.byref(make_desc(d)), ctypes.byref(b), None)
    if n < 0:
        raise NtcError(NTC_ERR_INVALID_ARGUMENT, lib().ntc_last_error().decode())
    boxes = np.zeros((n, 6), np.int32)
    lib().ntc_train_footprint(ctypes.byref(make_desc(d)), ctypes.byref(b), boxes.ctypes.data_as(ctypes.c_void_p))
    return boxes


def _b(batch):
    return batch[0] if isinstance(batch, tuple) else batch


def ntc_footprint_size(d, batch) -> int:
    n = lib().ntc_footprint_size(ctypes.byref(make_desc(d)), ctypes.byref(_b(batch)))
    if n < 0:
        raise NtcError(NTC_ERR_INVALID_ARGUMENT, lib().ntc_last_error().decode())
    return n


def ntc_footprint_pack(d, batch, src: torch.Tensor, packed: torch.Tensor, stream=None):
    _check(lib().ntc_footprint_pack(ctypes.byref(make_desc(d)), ctypes.byref(_b(batch)), _ptr(src), _ptr(packed),
                                    _stream(stream)))


NTC_BOX_PACK, NTC_BOX_UNPACK, NTC_BOX_ADD, NTC_BOX_ZERO = 0, 1, 2, 3


def _boxes_arg(boxes):
    import numpy as np

    bx = np.ascontiguousarray(np.asarray(boxes, dtype=np.int32).reshape(-1, 6))
    return bx, bx.ctypes.data_as(ctypes.c_void_p), bx.shape[0]


def ntc_boxes_size(d, boxes) -> int:
    bx, ptr, n = _boxes_arg(boxes)
    v = lib().ntc_boxes_size(ctypes.byref(make_desc(d)), ptr, n)
    if v < 0:
        raise NtcError(NTC_ERR_INVALID_ARGUMENT, lib().ntc_last_error().decode())
    return int(v)


def ntc_boxes_copy(d, boxes, src, dst: torch.Tensor, mode: int, stream=None):
    bx, ptr, n = _boxes_arg(boxes)
    _check(lib().ntc_boxes_copy(ctypes.byref(make_desc(d)), ptr, n, _ptr(src), _ptr(dst), mode, _stream(stream)))


def ntc_train_apply_boxes(trainer: Trainer, buffers: TrainBuffers, boxes, hp: Hparams, stream=None):
    bx, ptr, n = _boxes_arg(boxes)
    _check(lib().ntc_train_apply_boxes(trainer.handle, ctypes.byref(trainer.desc), ctypes.byref(buffers), ptr, n,
                                       ctypes.byref(hp), _stream(stream)))


def ntc_footprint_unpack(d, batch, packed, dst: torch.Tensor, stream=None):
    _check(lib().ntc_footprint_unpack(ctypes.byref(make_desc(d)), ctypes.byref(_b(batch)), _ptr(packed), _ptr(dst),
                                      _stream(stream)))
