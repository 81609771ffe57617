"""Host logic of the sharded data-parallel training mode (latent grids sharded by row bands,
SURVEY.md 8(e)), CPU only: band partition, crop ownership, the exchange plan (each rank's
footprint = its own-band part + the halo pieces fetched from the owners, exactly once), and
the variable-size all-to-all over a gloo group of 3 processes."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2305_17105_b200 as ntc
from paper_2305_17105_b200.dist import band, band_boxes, crop_owners, exchange_plan, grid_rows, intersect_band
from paper_2305_17105_b200.synth import Profile, gen_crops

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_bands_partition_every_grid(world):
    d = Profile.named("ntc0.2", 1024, 8)
    NL = ntc.ntc_num_latents(d)
    total = sum(ntc.ntc_boxes_size(d, band_boxes(d, world, r)) if band_boxes(d, world, r).size else 0
                for r in range(world))
    assert total == NL
    for j in range(ntc.ntc_num_levels(d)):
        for k in range(2):
            R = grid_rows(d, j, k)
            rows = np.concatenate([np.arange(*band(R, world, r)) for r in range(world)])
            assert np.array_equal(rows, np.arange(R))


@pytest.mark.parametrize("world,mip", [(2, 0), (3, 0), (4, 2), (8, 5)])
def test_exchange_plan_covers_footprints_once(world, mip):
    d = Profile.named("ntc0.2", 512, 8)
    g = gen_crops(11 + mip, 512, mip, 7, 64)
    own = crop_owners(d, mip, g, world)
    assert own.min() >= 0 and own.max() < world
    crops, need, plan = exchange_plan(d, mip, g, world)
    assert sum(c.shape[0] for c in crops) == g.shape[0]
    for s in range(world):
        if need[s].size == 0:
            continue
        own_part = intersect_band(d, need[s], world, s)
        parts = [own_part] + [plan[s][t] for t in range(world) if t != s]
        covered = sum(ntc.ntc_boxes_size(d, p) for p in parts if p.size)
        assert covered == ntc.ntc_boxes_size(d, need[s])
        for t in range(world):
            if plan[s][t].size:  # halo pieces lie in the sender's band
                lo, hi = zip(*[band(grid_rows(d, int(b[0]), int(b[1])), world, t) for b in plan[s][t]])
                assert np.all(plan[s][t][:, 3] >= np.array(lo)) and np.all(plan[s][t][:, 5] < np.array(hi))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys

    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2305_17105_b200.dist import _all_to_all

        # rank r sends (r*10 + t) repeated (r + t + 1) times to rank t
        send = [torch.full((rank + t + 1,), float(rank * 10 + t)) for t in range(world)]
        recv = _all_to_all(dist, None, send, [s + rank + 1 for s in range(world)], torch.device("cpu"))
        ok = all(torch.equal(recv[s], torch.full((s + rank + 1,), float(s * 10 + rank))) for s in range(world))
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


def test_all_to_all_variable_sizes_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 3, port, q)) for r in range(3)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(3)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok in res)


def test_stacked_segments_layout():
    """C5 batched exchange (StackedDataParallelTrainer): per peer, the materials' pieces are
    contiguous and in material order; offsets tile the send and receive buffers exactly."""
    from paper_2305_17105_b200.dist import StepPlan, stacked_segments

    d = Profile.named("ntc0.2", 512, 8)
    world = 3
    for rank in range(world):
        plans = [StepPlan(d, 3, gen_crops(30 + k, 512, 3, 6, 32), world, rank) for k in range(4)]
        ssz, rsz, soff, roff = stacked_segments(plans)
        assert ssz == [sum(p.send_sizes[t] for p in plans) for t in range(world)]
        assert rsz == [sum(p.recv_sizes[t] for p in plans) for t in range(world)]
        pos_s = pos_r = 0
        for t in range(world):
            for k, p in enumerate(plans):
                assert soff[k][t] == pos_s and roff[k][t] == pos_r
                pos_s += p.send_sizes[t]
                pos_r += p.recv_sizes[t]
        assert pos_s == sum(ssz) and pos_r == sum(rsz)


def _stacked_worker(rank, world, port, q):
    """The batched all-to-all of several materials' halo pieces over gloo (host tensors): what
    rank s receives from t for material k is exactly what t packed for s for material k."""
    import sys

    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2305_17105_b200.dist import StepPlan, _all_to_all, stacked_segments

        d = Profile.named("ntc0.2", 512, 8)
        plans = [StepPlan(d, 4, gen_crops(50 + k, 512, 4, 6, 16), world, rank) for k in range(3)]
        ssz, rsz, soff, roff = stacked_segments(plans)
        send = torch.zeros(sum(ssz))
        for k, p in enumerate(plans):  # piece (k -> t) filled with a code of (sender, k, t)
            for t in range(world):
                send[soff[k][t]: soff[k][t] + p.send_sizes[t]] = 1000 * rank + 100 * k + t
        pieces = list(torch.split(send, ssz))
        recv = torch.cat(_all_to_all(dist, None, pieces, rsz, torch.device("cpu")))
        ok = True
        for k, p in enumerate(plans):
            for t in range(world):
                seg = recv[roff[k][t]: roff[k][t] + p.recv_sizes[t]]
                ok &= bool(torch.all(seg == 1000 * t + 100 * k + rank))
        q.put((rank, ok, sum(rsz)))
    finally:
        dist.destroy_process_group()


def test_stacked_exchange_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_stacked_worker, args=(r, 3, port, q)) for r in range(3)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(3)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok, _ in res)
    assert sum(n for _, _, n in res) > 0  # the crops at mip 4 do read other bands
