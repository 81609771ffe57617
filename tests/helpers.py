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
