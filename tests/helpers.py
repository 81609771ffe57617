"""Shared test helpers: seeded materials for both the CUDA path and the oracle."""
from __future__ import annotations

import numpy as np

from paper_2305_17105_b200.synth import Profile, gen_codes, gen_weights_f16


def oracle_grid_list(O, d):
    out = []
    for j in range(O.num_levels(d)):
        r0, r1 = O.grid_res(d, j)
        out += [(r0 * r0 * d.c0, d.b0), (r1 * r1 * d.c1, d.b1)]
    return out


def material_inputs(O, d: Profile, seed: int, out_gain: float = 0.3):
    codes = gen_codes(seed, oracle_grid_list(O, d))
    w = gen_weights_f16(seed + 1, d.input_dim, d.channels, d.hidden_mats, out_gain)
    return codes, w


def chain_queries(W: int, mips, stride: int = 1):
    q = []
    for m in mips:
        wm = W >> m
        ys, xs = np.meshgrid(np.arange(0, wm, stride), np.arange(0, wm, stride), indexing="ij")
        q.append(np.stack([xs.ravel(), ys.ravel(), np.full(xs.size, m)], 1))
    return np.concatenate(q).astype(np.int32)


def oracle_footprint(O, d, mip, crops):
    """Latents the crops' texels read at `mip`, from the oracle's addressing (ntco_address):
    the footprint-sparse Adam domain (R18)."""
    fp = np.zeros(O.num_latents(d), bool)
    for x0, y0, w, h in np.asarray(crops).reshape(-1, 4):
        for y in range(y0, y0 + h):
            for x in range(x0, x0 + w):
                ti, _ = O.address(d, mip, x, y)
                r0, r1 = O.grid_res(d, ti[0])
                for t in range(4):
                    a = O.grid_offset(d, ti[0], 0) + (ti[2 + 2 * t] * r0 + ti[1 + 2 * t]) * d.c0
                    fp[a: a + d.c0] = True
                    b = O.grid_offset(d, ti[0], 1) + (ti[10 + 2 * t] * r1 + ti[9 + 2 * t]) * d.c1
                    fp[b: b + d.c1] = True
    return fp


def grid_spans(O, d):
    """[(slice, bits)] of every grid in the canonical latent array."""
    out = []
    for j in range(O.num_levels(d)):
        for k, B in ((0, d.b0), (1, d.b1)):
            a = O.grid_offset(d, j, k)
            b = O.grid_offset(d, j, 1) if k == 0 else O.grid_offset(d, j + 1, 0)
            out.append((slice(a, b), B))
    return out


def centres(O, d, codes):
    """Bin centres (code - (N/2 - 1)) Q of every grid's codes."""
    lat = np.zeros(codes.shape, np.float32)
    for sl, B in grid_spans(O, d):
        lat[sl] = (codes[sl].astype(np.float64) - (2**B // 2 - 1)) / 2**B
    return lat
