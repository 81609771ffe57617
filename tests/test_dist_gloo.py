"""Multi-process (world_size 2, gloo, CPU) checks of the data-parallel training decomposition:
the round-robin crop split covers the global batch exactly once, and the sum over ranks of
the per-rank gradients (loss normalised by the global batch) all-reduced through
torch.distributed equals the global-batch gradient -- computed here with the CPU oracle."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


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
        import oracle as O
        from paper_2305_17105_b200.dist import crop_texels, split_crops
        from paper_2305_17105_b200.synth import (Profile, box_mip_chain_u8, gen_crops, gen_latents,
                                                 gen_reference_u8, gen_weights_f32, u8_to_f16_bits)

        d = Profile.named("ntc0.2", 64, 4)
        lat = gen_latents(1, O.num_latents(d))
        par = gen_weights_f32(2, d.input_dim, 4, out_gain=1.0)
        ref = u8_to_f16_bits(box_mip_chain_u8(gen_reference_u8(3, 64, 4))[1])
        gcrops = gen_crops(4, 64, 1, 5, 12)  # 5 crops: ranks get 3 and 2
        mine = split_crops(gcrops, world, rank)
        # every global crop is owned by exactly one rank
        owned = torch.zeros(len(gcrops), dtype=torch.int64)
        owned[rank::world] = 1
        dist.all_reduce(owned)
        assert torch.all(owned == 1)
        Bg, Bm = crop_texels(gcrops), crop_texels(mine)
        loss, dp, dl = O.train_grads(d, lat, par, 1, mine, ref, 9, 2)
        s = Bm / Bg  # rescale the oracle's own-batch mean to the global-batch normalisation
        flat = torch.from_numpy(np.concatenate([dp * s, [loss * s], dl * s]))
        dist.all_reduce(flat)
        if rank == 0:
            lg, dpg, dlg = O.train_grads(d, lat, par, 1, gcrops, ref, 9, 2)
            f = flat.numpy()
            P = dp.size
            ok = (abs(f[P] - lg) <= 1e-12 * lg and np.allclose(f[:P], dpg, rtol=1e-10, atol=1e-15)
                  and np.allclose(f[P + 1:], dlg, rtol=1e-10, atol=1e-15))
            q.put(bool(ok))
    finally:
        dist.destroy_process_group()


def test_dp_gradient_decomposition_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    assert q.get(timeout=10) is True
