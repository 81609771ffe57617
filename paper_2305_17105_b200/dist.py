"""Multi-GPU plumbing (one process per GPU, torch.distributed for the collectives).

Decode: no exchange is needed.  Independent materials go to
independent ranks (material-parallel, weak scaling); one material's chain is split into
equal contiguous tile ranges with ntc_decode_chain_part.

Training, data-parallel over texel batches: every rank holds the (small) model replicated
-- latents 49 MB and 8,457 weights at 4096^2 NTC 0.2 -- and the same global crop list (same
seed).  Rank r trains on crops r, r+N, ... with the loss normalised by the GLOBAL batch
(ntc_batch.norm_texels), so the sum of the ranks' gradients is the global gradient.  One
all-reduce (NCCL over NVLink) exchanges [dW | loss | latent gradients packed over the global
batch footprint]; every rank then applies the identical Adam step over the global
footprint, keeping the replicas bit-identical.
"""
from __future__ import annotations

import numpy as np
import torch

from . import (NTC_STEP_APPLY, NTC_STEP_GRADS, Hparams, Trainer, make_batch, make_buffers, ntc_footprint_pack,
               ntc_footprint_size, ntc_footprint_unpack, ntc_num_latents, ntc_num_params, ntc_train_step)


def split_crops(global_crops, world: int, rank: int) -> np.ndarray:
    """Crops of this rank: global crops rank, rank + world, ... (round robin)."""
    g = np.asarray(global_crops, np.int32).reshape(-1, 4)
    return np.ascontiguousarray(g[rank::world])


def crop_texels(crops) -> int:
    c = np.asarray(crops, np.int64).reshape(-1, 4)
    return int((c[:, 2] * c[:, 3]).sum())


class DataParallelTrainer:
    """Replicated NTC training state on one rank + the per-step gradient exchange."""

    def __init__(self, d, latents: torch.Tensor, params: torch.Tensor, group=None):
        import torch.distributed as dist

        self.d = d
        self.group = group
        self.dist = dist if dist.is_initialized() else None
        self.world = dist.get_world_size(group) if self.dist else 1
        self.rank = dist.get_rank(group) if self.dist else 0
        dev = latents.device
        NL, P = ntc_num_latents(d), ntc_num_params(d)
        assert latents.numel() == NL and params.numel() == P
        self.P = P
        self.t = {"latents": latents, "params": params}
        for k in ("m_lat", "v_lat", "grad_lat", "noisy"):
            self.t[k] = torch.zeros(NL, device=dev)
        for k in ("m_par", "v_par"):
            self.t[k] = torch.zeros(P, device=dev)
        if self.dist and self.world > 1:  # replicas start identical
            self.dist.broadcast(self.t["latents"], 0, group=group)
            self.dist.broadcast(self.t["params"], 0, group=group)
        self.flat = torch.zeros(P + 1, device=dev)
        self.trainer = Trainer(d)
        self.loss = None

    def _flat(self, n):
        if self.flat.numel() < self.P + 1 + n:
            self.flat = torch.zeros(self.P + 1 + n, device=self.flat.device)
        return self.flat[: self.P + 1 + n]

    def step(self, mip: int, global_crops, ref: torch.Tensor, ref_stride: int, hp: Hparams) -> torch.Tensor:
        d = self.d
        gcrops = np.asarray(global_crops, np.int32).reshape(-1, 4)
        mine = split_crops(gcrops, self.world, self.rank)
        gbatch = make_batch(mip, gcrops, ref, ref_stride)
        nfp = ntc_footprint_size(d, gbatch)
        flat = self._flat(nfp)
        grad_par, loss, packed = flat[: self.P], flat[self.P: self.P + 1], flat[self.P + 1:]
        self.t["grad_par"] = grad_par
        bufs = make_buffers(self.t)
        # zero the global footprint, then this rank's crops (loss normalised by the global batch)
        ntc_footprint_unpack(d, gbatch, None, self.t["grad_lat"])
        if mine.shape[0] > 0:
            mb = make_batch(mip, mine, ref, ref_stride, norm_texels=crop_texels(gcrops))
            ntc_train_step(self.trainer, bufs, mb, hp, loss, flags=NTC_STEP_GRADS)
        else:
            flat[: self.P + 1].zero_()
        ntc_footprint_pack(d, gbatch, self.t["grad_lat"], packed)
        if self.dist and self.world > 1:
            self.dist.all_reduce(flat, group=self.group)  # one collective: [dW | loss | dLatent]
        ntc_footprint_unpack(d, gbatch, packed, self.t["grad_lat"])
        ntc_train_step(self.trainer, bufs, gbatch, hp, loss, flags=NTC_STEP_APPLY)
        self.loss = loss
        return loss
