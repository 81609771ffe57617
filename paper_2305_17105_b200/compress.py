"""The compression loop around ntc_train_step (PAPER.md:420-431,
509-534, 564-575).  Host-side scheduling only; every step runs in the CUDA library.

- per batch one LOD: LOD = floor(-log4 X), X ~ U(0,1), clamped to the chain; 5% of the
  batches draw the LOD uniformly over the chain;
- crops of min(crop, mip width) at uniform positions (R19), `crops` per batch;
- learning rates 0.01 (latents) / 0.005 (weights) with cosine annealing to 0 over the whole
  run, Adam;
- simulated quantisation noise, clamp after each update;
- at the end: explicit quantisation, latents frozen at their bin centres, and 5% more steps
  that optimise only the weights.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import (NTC_STEP_APPLY, NTC_STEP_GRADS, Hparams, Trainer, make_batch, make_buffers, ntc_dequantize_codes,
               ntc_grid_layout, ntc_num_latents, ntc_num_levels, ntc_num_mips, ntc_num_params, ntc_quantize_latents,
               ntc_train_step)


def sample_lod(rng: np.random.Generator, num_mips: int, uniform_fraction: float = 0.05) -> int:
    """LOD = floor(-log4 X), X ~ U(0,1] (clamped to the chain); with
    probability `uniform_fraction` the LOD is uniform over the chain instead."""
    if rng.random() < uniform_fraction:
        return int(rng.integers(0, num_mips))
    x = 1.0 - rng.random()  # (0, 1]
    return min(int(math.floor(-math.log(x, 4.0))), num_mips - 1)


def lr_at(step: int, total: int, lr0: float) -> float:
    """Cosine annealing from lr0 to 0 over `total` steps."""
    return lr0 * 0.5 * (1.0 + math.cos(math.pi * step / total))


@dataclass
class CompressConfig:
    steps: int = 250_000
    finetune_fraction: float = 0.05
    crops: int = 8
    crop: int = 256
    lr_latent: float = 0.01
    lr_weight: float = 0.005
    uniform_lod_fraction: float = 0.05
    seed: int = 0


def init_state(d, seed: int, device):
    """Latents uniform over the central 50% of each grid's quantisation range, weights
    He-uniform (fan-in), biases zero (the paper states neither)."""
    rng = np.random.default_rng(seed)
    lat = np.zeros(ntc_num_latents(d), np.float32)
    for j in range(ntc_num_levels(d)):
        r0, r1, o0, o1 = ntc_grid_layout(d, j)
        for off, n, B in ((o0, r0 * r0 * d.c0, d.b0), (o1, r1 * r1 * d.c1, d.b1)):
            N = 2**B
            lo, hi = -(N - 1) / 2 / N, N / 2 / N
            mid, half = (lo + hi) / 2, (hi - lo) / 4
            lat[off: off + n] = rng.uniform(mid - half, mid + half, n)
    D = 4 * d.c0 + d.c1 + 13
    dims = [(D, 64)] + [(64, 64)] * d.hidden_mats + [(64, d.channels)]
    par = []
    for fi, fo in dims:
        b = math.sqrt(6.0 / fi)
        par += [rng.uniform(-b, b, fi * fo), np.zeros(fo)]
    par = np.concatenate(par).astype(np.float32)
    assert par.size == ntc_num_params(d)
    return torch.from_numpy(lat).to(device), torch.from_numpy(par).to(device)


class Compressor:
    """Trains one material against its reference mip chain (fp16 device tensors, (h, w, c))."""

    def __init__(self, d, ref_chain, cfg: CompressConfig, device="cuda"):
        self.d, self.cfg, self.ref = d, cfg, ref_chain
        assert len(ref_chain) == ntc_num_mips(d)
        lat, par = init_state(d, cfg.seed, device)
        NL, P = ntc_num_latents(d), ntc_num_params(d)
        self.t = {"latents": lat, "params": par}
        for k in ("m_lat", "v_lat", "grad_lat", "noisy"):
            self.t[k] = torch.zeros(NL, device=device)
        for k in ("m_par", "v_par", "grad_par"):
            self.t[k] = torch.zeros(P, device=device)
        self.buf = make_buffers(self.t)
        self.trainer = Trainer(d)
        self.loss = torch.zeros(1, device=device)
        self.status = torch.zeros(1, dtype=torch.int32, device=device)
        self.rng = np.random.default_rng(cfg.seed + 1)
        self.codes = torch.empty(NL, dtype=torch.uint8, device=device)
        self.step_no = 0
        self.total = int(round(cfg.steps * (1.0 + cfg.finetune_fraction)))
        self.losses = []

    def _batch(self):
        d, cfg = self.d, self.cfg
        M = ntc_num_mips(d)
        m = sample_lod(self.rng, M, cfg.uniform_lod_fraction)
        wm = d.width >> m
        cs = min(cfg.crop, wm)
        x0 = self.rng.integers(0, wm - cs + 1, cfg.crops)
        y0 = self.rng.integers(0, wm - cs + 1, cfg.crops)
        crops = np.stack([x0, y0, np.full(cfg.crops, cs), np.full(cfg.crops, cs)], 1).astype(np.int32)
        return make_batch(m, crops, self.ref[m], wm * d.channels)

    def plan(self, frozen: bool):
        """The next step's batch and hyper-parameters: LOD + crops, cosine
        learning rates; noise on and latents trained in the noisy phase, noise
        off and latents frozen after the explicit quantisation (R25)."""
        cfg = self.cfg
        self.step_no += 1
        t = self.step_no
        hp = Hparams(lr_at(t - 1, self.total, cfg.lr_latent), lr_at(t - 1, self.total, cfg.lr_weight), 0.9, 0.999,
                     1e-8, t, cfg.seed, 0 if frozen else 1, 0, 1 if frozen else 0)
        return self._batch(), hp

    def step(self, frozen: bool, record: bool = False):
        batch, hp = self.plan(frozen)
        ntc_train_step(self.trainer, self.buf, batch, hp, self.loss, self.status,
                       flags=NTC_STEP_GRADS | NTC_STEP_APPLY)
        if record:
            self.losses.append((self.step_no, float(self.loss.item())))

    def freeze(self):
        """Explicit quantisation; latents become their bin centres."""
        ntc_quantize_latents(self.d, self.t["latents"], self.codes)
        ntc_dequantize_codes(self.d, self.codes, self.t["latents"])

    def run(self, log_every: int = 0):
        S = self.cfg.steps
        for i in range(S):
            self.step(False, record=bool(log_every) and (i % log_every == 0))
        self.freeze()
        for i in range(self.total - S):
            self.step(True, record=bool(log_every) and (i % log_every == 0))
        if int(self.status.item()) != 0:
            raise FloatingPointError("non-finite loss during compression (SPEC.md:278)")
        return self.codes, self.t["params"].to(torch.float16)
