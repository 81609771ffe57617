"""Seeded synthetic inputs shared by the tests, the oracle leg and the bench.

This module holds NONE of the method's arithmetic (no quantisation, addressing,
encoding or network code): it only draws random numbers of the shapes and value
distributions described in DESIGN.md "Input recipe".  Grid sizes are passed in by
the caller (from the product library's or the oracle's own geometry).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

# Table 2: (g0_ratio, C0, B0, C1, B1)
PROFILES = {
    "ntc0.2": (4, 8, 2, 12, 4),
    "ntc0.5": (4, 12, 4, 20, 4),
    "ntc1.0": (2, 12, 2, 10, 4),
    "ntc2.25": (2, 16, 4, 12, 4),
}

SEED_BASE = 0x4E544300  # per-config seed = SEED_BASE + config index


@dataclass(frozen=True)
class Profile:
    width: int
    channels: int
    g0_ratio: int = 4
    c0: int = 8
    b0: int = 2
    c1: int = 12
    b1: int = 4
    hidden_mats: int = 1
    activation: int = 0

    @staticmethod
    def named(name: str, width: int, channels: int, hidden_mats: int = 1, activation: int = 0) -> "Profile":
        r, c0, b0, c1, b1 = PROFILES[name]
        return Profile(width, channels, r, c0, b0, c1, b1, hidden_mats, activation)

    @property
    def input_dim(self) -> int:  # PAPER.md:493 (shape bookkeeping only)
        return 4 * self.c0 + self.c1 + 13


def gen_codes(seed: int, grids) -> np.ndarray:
    """grids: iterable of (n_values, bits).  iid uniform codes in [0, 2^bits - 1],
    concatenated in the given order (uint8)."""
    rng = np.random.default_rng(seed)
    parts = [rng.integers(0, 1 << b, size=n, dtype=np.uint8) for n, b in grids]
    return np.concatenate(parts) if parts else np.zeros(0, np.uint8)


def gen_latents(seed: int, n: int, scale: float = 0.2) -> np.ndarray:
    """fp32 training latents ~ U(-scale, scale) (inside every profile's quant range)."""
    rng = np.random.default_rng(seed)
    return rng.uniform(-scale, scale, size=n).astype(np.float32)


def _weights_f64(seed: int, D: int, c: int, hidden_mats: int, out_gain: float) -> np.ndarray:
    rng = np.random.default_rng(seed)
    H = 64
    parts = []
    dims = [(D, H)] + [(H, H)] * hidden_mats + [(H, c)]
    for li, (fi, fo) in enumerate(dims):
        last = li == len(dims) - 1
        bound = np.sqrt(6.0 / fi) * (out_gain if last else 1.0)
        parts.append(rng.uniform(-bound, bound, size=fo * fi))
        if last:
            parts.append(0.5 + rng.uniform(-0.1, 0.1, size=fo))
        else:
            parts.append(rng.uniform(-0.1, 0.1, size=fo))
    return np.concatenate(parts)


def gen_weights_f16(seed: int, D: int, c: int, hidden_mats: int = 1, out_gain: float = 0.3) -> np.ndarray:
    """MLP weights in the ABI order W1[64][D], b1, W2[64][64], b2, [W2b, b2b], W3[c][64], b3,
    as fp16 bit patterns (uint16).  He-uniform hidden layers, output gain `out_gain`."""
    w = _weights_f64(seed, D, c, hidden_mats, out_gain)
    return w.astype(np.float16).view(np.uint16)


def gen_weights_f32(seed: int, D: int, c: int, hidden_mats: int = 1, out_gain: float = 0.3) -> np.ndarray:
    return _weights_f64(seed, D, c, hidden_mats, out_gain).astype(np.float32)


def _smooth_field(rng, n: int, octaves: int = 4) -> np.ndarray:
    y = np.arange(n, dtype=np.float32)[:, None] / n
    x = np.arange(n, dtype=np.float32)[None, :] / n
    f = np.zeros((n, n), np.float32)
    for o in range(octaves):
        fr = 2.0 ** (o + 1)
        for _ in range(2):
            a = rng.uniform(0, 2 * np.pi, 4).astype(np.float32)
            k = rng.uniform(0.5, 1.5, 2).astype(np.float32) * fr
            f += (np.sin(2 * np.pi * k[0] * x + a[0]) * np.cos(2 * np.pi * k[1] * y + a[1])) / (o + 1)
    f -= f.min()
    f /= max(float(f.max()), 1e-6)
    return f


def gen_reference_u8(seed: int, width: int, channels: int) -> np.ndarray:
    """Mip-0 reference texture set (width, width, c) unorm8: c correlated channels, a
    rank-3 mix of 3 smooth fields plus 10% independent noise (motivated by Fig 2)."""
    rng = np.random.default_rng(seed)
    fields = np.stack([_smooth_field(rng, width) for _ in range(3)], -1)  # (w, w, 3)
    mix = rng.uniform(0.0, 1.0, size=(3, channels)).astype(np.float32)
    mix /= mix.sum(0, keepdims=True)
    img = fields @ mix
    img = 0.9 * img + 0.1 * rng.uniform(0.0, 1.0, size=img.shape).astype(np.float32)
    return np.clip(np.rint(img * 255.0), 0, 255).astype(np.uint8)


def box_mip_chain_u8(img: np.ndarray):
    """Box-filtered mip chain of a (w, w, c) unorm8 image down to 1x1 (data generation)."""
    chain = [img]
    cur = img.astype(np.float32)
    while cur.shape[0] > 1:
        cur = 0.25 * (cur[0::2, 0::2] + cur[1::2, 0::2] + cur[0::2, 1::2] + cur[1::2, 1::2])
        chain.append(np.clip(np.rint(cur), 0, 255).astype(np.uint8))
    return chain


def u8_to_f16_bits(img_u8: np.ndarray) -> np.ndarray:
    """R24: reference texels R = fp16(v / 255), computed once on the host."""
    return (img_u8.astype(np.float64) / 255.0).astype(np.float16).view(np.uint16)


def gen_queries(seed: int, width: int, n: int, mode: str = "area") -> np.ndarray:
    """Random texel queries (n, 3) int32 (x, y, mip) over a width^2 mip chain.
    mode 'area': uniform over the chain's texels; 'mip': mip uniform, then (x, y)."""
    rng = np.random.default_rng(seed)
    M = int(np.log2(width)) + 1
    sizes = np.array([(width >> m) ** 2 for m in range(M)], np.int64)
    if mode == "area":
        g = rng.integers(0, int(sizes.sum()), size=n, dtype=np.int64)
        starts = np.concatenate([[0], np.cumsum(sizes)])
        mip = np.searchsorted(starts, g, side="right") - 1
        r = g - starts[mip]
    else:
        mip = rng.integers(0, M, size=n, dtype=np.int64)
        r = (rng.random(n) * sizes[mip]).astype(np.int64)
    wm = width >> mip
    return np.stack([r % wm, r // wm, mip], 1).astype(np.int32)


def gen_crops(seed: int, width: int, mip: int, n_crops: int, crop: int = 256) -> np.ndarray:
    """R19: crop origins uniform over valid positions, size min(crop, mip dim)."""
    rng = np.random.default_rng(seed)
    wm = width >> mip
    cs = min(crop, wm)
    x0 = rng.integers(0, wm - cs + 1, size=n_crops)
    y0 = rng.integers(0, wm - cs + 1, size=n_crops)
    return np.stack([x0, y0, np.full(n_crops, cs), np.full(n_crops, cs)], 1).astype(np.int32)


def gen_grads(seed: int, n: int, scale: float = 1e-3, zero_frac: float = 0.3) -> np.ndarray:
    """Synthetic fp32 gradients (for isolated optimizer parity), some exactly zero."""
    rng = np.random.default_rng(seed)
    g = rng.normal(0.0, scale, size=n).astype(np.float32)
    g[rng.random(n) < zero_frac] = 0.0
    return g
