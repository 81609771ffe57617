"""Multi-GPU plumbing (one process per GPU, torch.distributed for the collectives).

Decode: no exchange is needed.  Independent materials go to
independent ranks (material-parallel, weak scaling); one material's chain is split into
equal contiguous tile ranges with ntc_decode_chain_part.

Training, data-parallel over texel batches, two modes:

- DataParallelTrainer (replicated latents): every rank holds the whole model -- latents 49 MB
  and 8,457 weights at 4096^2 NTC 0.2 -- and the same global crop list (same seed).  Rank r
  trains on crops r, r+N, ... with the loss normalised by the GLOBAL batch
  (ntc_batch.norm_texels), so the sum of the ranks' gradients is the global gradient.  One
  all-reduce (NCCL over NVLink) exchanges [dW | loss | latent gradients packed over the
  global batch footprint]; every rank then applies the identical Adam step over the global
  footprint, keeping the replicas bit-identical.
- ShardedDataParallelTrainer (latent grids sharded by tile): rank r OWNS a
  row band of every latent grid -- the authoritative latents and their Adam state.  Crops go
  to the owner of their origin's G0 row.  Per step: the halo latents a rank's crops read in
  other bands are fetched from their owners (one all-to-all of packed boxes), GRADS runs on
  the rank's crops, the latent gradients that fall in other bands go back to their owners
  (the reverse all-to-all, added there), [dW | loss] is all-reduced, and every owner applies
  Adam + clamp to its band of the global footprint (weights redundantly everywhere).
"""
from __future__ import annotations

import numpy as np
import torch

from . import (NTC_BOX_ADD, NTC_BOX_PACK, NTC_BOX_UNPACK, NTC_BOX_ZERO, NTC_STEP_APPLY, NTC_STEP_GRADS, Hparams,
               Trainer, make_batch, make_buffers, ntc_boxes_copy, ntc_boxes_size, ntc_footprint_pack,
               ntc_footprint_size, ntc_footprint_unpack, ntc_grid_layout, ntc_level_of_mip, ntc_num_latents,
               ntc_num_levels, ntc_num_params, ntc_train_apply_boxes, ntc_train_footprint, ntc_train_step)


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


# ------------------------------------------------------------------ sharded latents
def band(rows: int, world: int, rank: int):
    """Row band [lo, hi) of a grid with `rows` rows owned by `rank`."""
    return rows * rank // world, rows * (rank + 1) // world


def grid_rows(d, level: int, k: int) -> int:
    r0, r1, _, _ = ntc_grid_layout(d, level)
    return r0 if k == 0 else r1


def owner_of_row(rows: int, world: int, y: int) -> int:
    for r in range(world):
        lo, hi = band(rows, world, r)
        if lo <= y < hi:
            return r
    return world - 1


def crop_owners(d, mip: int, crops, world: int) -> np.ndarray:
    """Owner rank of each crop: the owner of the G0 row its origin texel reads (tap row of
    R1-R3, integer form), at the batch's feature level."""
    c = np.asarray(crops, np.int64).reshape(-1, 4)
    j = ntc_level_of_mip(d, mip)
    r0 = grid_rows(d, j, 0)
    w = d.width >> mip
    out = np.zeros(c.shape[0], np.int64)
    for i, (_, y0, _, _) in enumerate(c):
        ty = max(((2 * int(y0) + 1) * r0 - w) // (2 * w), 0)  # floor((y + 1/2) r0 / w - 1/2)
        out[i] = owner_of_row(r0, world, min(ty, r0 - 1))
    return out


def intersect_band(d, boxes, world: int, rank: int) -> np.ndarray:
    """Footprint boxes (level, k, x0, y0, x1, y1) clipped to `rank`'s row band of their grid."""
    out = []
    for lv, k, x0, y0, x1, y1 in np.asarray(boxes, np.int64).reshape(-1, 6):
        lo, hi = band(grid_rows(d, int(lv), int(k)), world, rank)
        a, b = max(int(y0), lo), min(int(y1), hi - 1)
        if a <= b:
            out.append((lv, k, x0, a, x1, b))
    return np.asarray(out, np.int32).reshape(-1, 6)


def band_boxes(d, world: int, rank: int) -> np.ndarray:
    """Every grid's full row band of `rank`."""
    out = []
    for j in range(ntc_num_levels(d)):
        for k in range(2):
            R = grid_rows(d, j, k)
            lo, hi = band(R, world, rank)
            if lo < hi:
                out.append((j, k, 0, lo, R - 1, hi - 1))
    return np.asarray(out, np.int32).reshape(-1, 6)


def stratified_crops(d, mip: int, world: int, per_rank: int, crop: int, rng) -> np.ndarray:
    """A global crop list with `per_rank` crops drawn uniformly inside every rank's row band
    (x uniform over the mip), so owner-based assignment is balanced: a stratified version of
    the uniform crop placement of R19 (each band gets the same number of crops)."""
    j = ntc_level_of_mip(d, mip)
    r0 = grid_rows(d, j, 0)
    w = d.width >> mip
    cs = min(crop, w)
    out = []
    for r in range(world):
        lo, hi = band(r0, world, r)
        ylo, yhi = (lo * w) // r0, (hi * w) // r0  # texel rows whose G0 tap row is in the band
        for _ in range(per_rank):
            a, b = ylo, max(ylo, min(yhi, w) - cs)
            y0 = int(rng.integers(min(a, w - cs), min(b, w - cs) + 1))
            x0 = int(rng.integers(0, w - cs + 1))
            out.append((x0, y0, cs, cs))
    return np.asarray(out, np.int32)


def exchange_plan(d, mip: int, global_crops, world: int):
    """For every rank s: its crops and the footprint boxes they read.  plan[s][t] = the boxes
    rank s reads inside rank t's band (what t sends to s); both sides derive the same plan."""
    g = np.asarray(global_crops, np.int32).reshape(-1, 4)
    own = crop_owners(d, mip, g, world)
    crops = [np.ascontiguousarray(g[own == s]) for s in range(world)]
    need = []
    for s in range(world):
        if crops[s].shape[0] == 0:
            need.append(np.zeros((0, 6), np.int32))
            continue
        need.append(ntc_train_footprint(d, make_batch(mip, crops[s], None, 0)))
    plan = [[intersect_band(d, need[s], world, t) if t != s else np.zeros((0, 6), np.int32) for t in range(world)]
            for s in range(world)]
    return crops, need, plan


def _all_to_all(dist, group, send, recv_sizes, dev):
    """Variable-size all-to-all of 1-D fp32 pieces (send[t] goes to rank t).  NCCL: one
    all_to_all_single on the device; gloo (tests): the same through host tensors."""
    inp = torch.cat([x.reshape(-1) for x in send]) if send else torch.zeros(0, device=dev)
    out_n = int(sum(recv_sizes))
    in_sizes = [int(x.numel()) for x in send]
    if dist.get_backend(group) == "nccl":
        out = torch.empty(out_n, device=dev)
        dist.all_to_all_single(out, inp, recv_sizes, in_sizes, group=group)
    else:
        out = torch.empty(out_n)
        dist.all_to_all_single(out, inp.cpu(), recv_sizes, in_sizes, group=group)
        out = out.to(dev)
    return list(torch.split(out, list(recv_sizes)))


class StepPlan:
    """Host-side schedule of one sharded step (pure function of the global crop list, so it
    can be built ahead of time, e.g. one step early or before a timed loop)."""

    def __init__(self, d, mip: int, global_crops, world: int, rank: int):
        g = np.asarray(global_crops, np.int32).reshape(-1, 4)
        crops, need, plan = exchange_plan(d, mip, g, world)
        self.mip = mip
        self.gcrops = g
        self.norm = crop_texels(g)
        self.mine = crops[rank]
        self.mine_g = intersect_band(d, ntc_train_footprint(d, make_batch(mip, g, None, 0)), world, rank)
        # halo latents this rank SENDS (to t: plan[t][rank]) and RECEIVES (from t: plan[rank][t]),
        # concatenated in rank order; the gradient exchange uses the same lists reversed
        self.send_boxes = [plan[t][rank] for t in range(world)]
        self.recv_boxes = [plan[rank][t] for t in range(world)]
        size = lambda bx: ntc_boxes_size(d, bx) if bx.size else 0  # noqa: E731
        self.send_sizes = [size(b) for b in self.send_boxes]
        self.recv_sizes = [size(b) for b in self.recv_boxes]
        self.send_all = _concat_boxes(self.send_boxes)
        self.recv_all = _concat_boxes(self.recv_boxes)
        # identical on every rank (derived from the global plan): skip the two all-to-alls
        # collectively when no rank reads outside its band (stratified crops usually do not)
        self.any_halo = any(plan[a][b].size for a in range(world) for b in range(world))


def _concat_boxes(lst):
    nz = [b for b in lst if b.size]
    return np.ascontiguousarray(np.concatenate(nz)) if nz else np.zeros((0, 6), np.int32)


class ShardedDataParallelTrainer:
    """Latent grids sharded by row bands; see the module docstring.  The
    device arrays keep the canonical full-size layout (the kernels address latents by their
    canonical index); only this rank's band is authoritative, the rest is a halo cache
    refreshed from the owners every step.  Per step: 5 box-copy launches at most (batched
    over all peers), GRADS (3), APPLY (1), two all-to-alls and one all-reduce."""

    MAXB = 256  # boxes per library call

    def __init__(self, d, latents: torch.Tensor, params: torch.Tensor, group=None):
        import torch.distributed as dist

        self.d, self.group = d, group
        self.dist = dist
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        dev = latents.device
        self.dev = dev
        NL, P = ntc_num_latents(d), ntc_num_params(d)
        assert latents.numel() == NL and params.numel() == P
        self.P = P
        self.t = {"latents": latents, "params": params}
        for k in ("m_lat", "v_lat", "grad_lat", "noisy"):
            self.t[k] = torch.zeros(NL, device=dev)
        for k in ("m_par", "v_par"):
            self.t[k] = torch.zeros(P, device=dev)
        self.dist.broadcast(self.t["params"], 0, group=group)  # weights replicated
        self.flat = torch.zeros(P + 1, device=dev)
        self.t["grad_par"] = self.flat[:P]
        self.trainer = Trainer(d)
        self.bufs = make_buffers(self.t)
        self.loss = None
        self.launches = 0  # library kernels launched by the last step (bench.py's gpu_launches)
        self._sbuf = torch.empty(0, device=dev)
        self._rbuf = torch.empty(0, device=dev)

    def plan(self, mip: int, global_crops) -> StepPlan:
        return StepPlan(self.d, mip, global_crops, self.world, self.rank)

    def _copy(self, bx, src, dst, mode):
        """Box copy in <= MAXB-box launches; packed operands advance with the boxes."""
        off = 0
        for i in range(0, bx.shape[0], self.MAXB):
            part = bx[i: i + self.MAXB]
            n = ntc_boxes_size(self.d, part)
            if mode == NTC_BOX_PACK:
                ntc_boxes_copy(self.d, part, src, dst[off: off + n], mode)
            elif mode == NTC_BOX_ZERO:
                ntc_boxes_copy(self.d, part, None, dst, mode)
            else:
                ntc_boxes_copy(self.d, part, src[off: off + n], dst, mode)
            off += n
            self.launches += 1

    def _buffers(self, ns, nr):
        if self._sbuf.numel() < ns:
            self._sbuf = torch.empty(ns, device=self.dev)
        if self._rbuf.numel() < nr:
            self._rbuf = torch.empty(nr, device=self.dev)
        return self._sbuf[:ns], self._rbuf[:nr]

    def _exchange(self, sbuf, ssizes, rbuf, rsizes):
        if self.dist.get_backend(self.group) == "nccl":
            self.dist.all_to_all_single(rbuf, sbuf, rsizes, ssizes, group=self.group)
        else:  # gloo (tests): through host memory
            out = torch.empty(rbuf.numel())
            self.dist.all_to_all_single(out, sbuf.cpu(), rsizes, ssizes, group=self.group)
            rbuf.copy_(out)

    def step(self, mip: int, global_crops, ref: torch.Tensor, ref_stride: int, hp: Hparams,
             plan: StepPlan = None) -> torch.Tensor:
        pl = plan if plan is not None else self.plan(mip, global_crops)
        self.launches = 0
        ns, nr = sum(pl.send_sizes), sum(pl.recv_sizes)
        sbuf, rbuf = self._buffers(ns, nr)
        # 1. halo latents from their owners (one batched pack, one all-to-all, one unpack)
        if pl.any_halo:
            self._copy(pl.send_all, self.t["latents"], sbuf, NTC_BOX_PACK)
            self._exchange(sbuf, pl.send_sizes, rbuf, pl.recv_sizes)
            self._copy(pl.recv_all, rbuf, self.t["latents"], NTC_BOX_UNPACK)
        # 2. zero this rank's share of the global footprint, then GRADS on its own crops
        self._copy(pl.mine_g, None, self.t["grad_lat"], NTC_BOX_ZERO)
        loss = self.flat[self.P: self.P + 1]
        if pl.mine.shape[0] > 0:
            mb = make_batch(pl.mip, pl.mine, ref, ref_stride, norm_texels=pl.norm)
            ntc_train_step(self.trainer, self.bufs, mb, hp, loss, flags=NTC_STEP_GRADS)
            self.launches += 3  # prep (+ weight image), fused forward/backward, reduce
        else:
            self.flat.zero_()
        # 3. halo gradients back to their owners (the reverse exchange), added there
        if pl.any_halo:
            self._copy(pl.recv_all, self.t["grad_lat"], rbuf, NTC_BOX_PACK)
            self._exchange(rbuf, pl.recv_sizes, sbuf, pl.send_sizes)
            self._copy(pl.send_all, sbuf, self.t["grad_lat"], NTC_BOX_ADD)
        # 4. [dW | loss] all-reduce; 5. owners apply Adam to their band of the global footprint
        self.dist.all_reduce(self.flat, group=self.group)
        ntc_train_apply_boxes(self.trainer, self.bufs, pl.mine_g, hp)
        self.launches += 1
        self.loss = loss
        return loss

    def gather_latents(self) -> torch.Tensor:
        """The full authoritative latent array on every rank (each owner's bands, all-gathered)."""
        d, N = self.d, self.world
        out = self.t["latents"].clone()
        mine = band_boxes(d, N, self.rank)
        buf = torch.empty(ntc_boxes_size(d, mine), device=self.dev)
        ntc_boxes_copy(d, mine, self.t["latents"], buf, NTC_BOX_PACK)
        sizes = [ntc_boxes_size(d, band_boxes(d, N, s)) for s in range(N)]
        recv = _all_to_all(self.dist, self.group, [buf] * N, sizes, self.dev)
        for s in range(N):
            if s != self.rank:
                ntc_boxes_copy(d, band_boxes(d, N, s), recv[s], out, NTC_BOX_UNPACK)
        return out


# ------------------------------------------------------------------ several materials (C5)
def stacked_segments(plans):
    """Layout of the batched halo exchange of several materials (C5): the
    piece a rank sends to peer t is [material 0 -> t | material 1 -> t | ...].  Returns
    (send_sizes[t], recv_sizes[t], send_off[k][t], recv_off[k][t]) where the offsets are
    positions inside the concatenated send / receive buffers (peer-major, then material)."""
    M = len(plans)
    world = len(plans[0].send_sizes) if M else 0
    send_sizes = [sum(p.send_sizes[t] for p in plans) for t in range(world)]
    recv_sizes = [sum(p.recv_sizes[t] for p in plans) for t in range(world)]
    send_off = [[0] * world for _ in range(M)]
    recv_off = [[0] * world for _ in range(M)]
    s = r = 0
    for t in range(world):
        for k in range(M):
            send_off[k][t], recv_off[k][t] = s, r
            s += plans[k].send_sizes[t]
            r += plans[k].recv_sizes[t]
    return send_sizes, recv_sizes, send_off, recv_off


class StackedDataParallelTrainer:
    """Several materials (C5: 64 x 4096^2) trained data-parallel over texel batches with the
    latent grids of every material sharded by row bands (ShardedDataParallelTrainer's
    scheme).  One step covers every material: ONE all-to-all carries all materials' halo
    latents, ONE the halo gradients back, and ONE all-reduce the stacked [dW | loss] of all
    materials ([M][P + 1] fp32: 64 x 33.8 KB = 2.2 MB at C5); owners then
    apply Adam to their bands.  Collectives per step: 3, independent of M."""

    def __init__(self, d, latents_list, params_list, group=None):
        import torch.distributed as dist

        self.d, self.group, self.dist = d, group, dist
        self.world, self.rank = dist.get_world_size(group), dist.get_rank(group)
        self.M = len(latents_list)
        dev = latents_list[0].device
        self.dev = dev
        self.P = ntc_num_params(d)
        self.stack = torch.zeros((self.M, self.P + 1), device=dev)  # [dW | loss] per material
        self.mats = []
        for k in range(self.M):
            tr = ShardedDataParallelTrainer(d, latents_list[k], params_list[k], group)
            tr.flat = self.stack[k]  # rows of the stacked all-reduce buffer
            tr.t["grad_par"] = tr.flat[: self.P]
            tr.bufs = make_buffers(tr.t)
            self.mats.append(tr)
        self._sbuf = torch.empty(0, device=dev)
        self._rbuf = torch.empty(0, device=dev)
        self.launches = 0

    def plan(self, mip: int, crops_list):
        """Per-material StepPlans and the batched exchange layout (host only, ahead of time)."""
        plans = [m.plan(mip, c) for m, c in zip(self.mats, crops_list)]
        return plans, stacked_segments(plans)

    def _buffers(self, ns, nr):
        if self._sbuf.numel() < ns:
            self._sbuf = torch.empty(ns, device=self.dev)
        if self._rbuf.numel() < nr:
            self._rbuf = torch.empty(nr, device=self.dev)
        return self._sbuf[:ns], self._rbuf[:nr]

    def step(self, mip: int, crops_list, refs, ref_stride: int, hp: Hparams, plan=None):
        """crops_list[k]: material k's global crop list; refs[k]: its reference mip image."""
        plans, (ssz, rsz, soff, roff) = plan if plan is not None else self.plan(mip, crops_list)
        self.launches = 0
        sbuf, rbuf = self._buffers(sum(ssz), sum(rsz))
        any_halo = any(p.any_halo for p in plans)
        # 1. every material's halo latents in one all-to-all
        if any_halo:
            for k, (m, pl) in enumerate(zip(self.mats, plans)):
                for t in range(self.world):
                    if pl.send_sizes[t]:
                        m._copy(pl.send_boxes[t], m.t["latents"], sbuf[soff[k][t]: soff[k][t] + pl.send_sizes[t]],
                                NTC_BOX_PACK)
            self.mats[0]._exchange(sbuf, ssz, rbuf, rsz)
            for k, (m, pl) in enumerate(zip(self.mats, plans)):
                for t in range(self.world):
                    if pl.recv_sizes[t]:
                        m._copy(pl.recv_boxes[t], rbuf[roff[k][t]: roff[k][t] + pl.recv_sizes[t]], m.t["latents"],
                                NTC_BOX_UNPACK)
        # 2. GRADS of every material on this rank's crops (rows of the stacked buffer)
        for m, pl, ref in zip(self.mats, plans, refs):
            m._copy(pl.mine_g, None, m.t["grad_lat"], NTC_BOX_ZERO)
            loss = m.flat[self.P: self.P + 1]
            if pl.mine.shape[0] > 0:
                mb = make_batch(pl.mip, pl.mine, ref, ref_stride, norm_texels=pl.norm)
                ntc_train_step(m.trainer, m.bufs, mb, hp, loss, flags=NTC_STEP_GRADS)
                m.launches += 3
            else:
                m.flat.zero_()
        # 3. every material's halo gradients back to their owners in one all-to-all
        if any_halo:
            for k, (m, pl) in enumerate(zip(self.mats, plans)):
                for t in range(self.world):
                    if pl.recv_sizes[t]:
                        m._copy(pl.recv_boxes[t], m.t["grad_lat"], rbuf[roff[k][t]: roff[k][t] + pl.recv_sizes[t]],
                                NTC_BOX_PACK)
            self.mats[0]._exchange(rbuf, rsz, sbuf, ssz)
            for k, (m, pl) in enumerate(zip(self.mats, plans)):
                for t in range(self.world):
                    if pl.send_sizes[t]:
                        m._copy(pl.send_boxes[t], sbuf[soff[k][t]: soff[k][t] + pl.send_sizes[t]], m.t["grad_lat"],
                                NTC_BOX_ADD)
        # 4. one all-reduce of the stacked [dW | loss]; 5. owners apply Adam per material
        self.dist.all_reduce(self.stack, group=self.group)
        for m, pl in zip(self.mats, plans):
            ntc_train_apply_boxes(m.trainer, m.bufs, pl.mine_g, hp)
            m.launches += 1
        self.launches = sum(m.launches for m in self.mats)
        return self.stack[:, self.P]

    def gather_latents(self, k: int) -> torch.Tensor:
        return self.mats[k].gather_latents()
