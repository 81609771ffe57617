"""GPU checks of the multi-GPU partitioner and the data-parallel training step.  Two ranks
share cuda:0 (this environment exposes one GPU) over a gloo group; the NCCL path is the same
code with backend="nccl" (bench.py under torchrun)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2305_17105_b200 as ntc
from paper_2305_17105_b200.synth import Profile
from helpers import material_inputs

pytestmark = pytest.mark.gpu
DEV = "cuda:0"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("nparts", [1, 2, 3, 8])
def test_decode_chain_part_covers_chain(O, nparts):
    """The union of the parts of ntc_decode_chain_part is bit-identical to ntc_decode_chain."""
    d = Profile.named("ntc0.2", 512, 9)
    codes, w = material_inputs(O, d, 5)
    mat = ntc.Material(d, torch.from_numpy(codes).to(DEV), torch.from_numpy(w.view(np.int16)).to(DEV))
    T = ntc.ntc_chain_texels(d)
    full = torch.empty(T * 9, dtype=torch.float16, device=DEV)
    ntc.ntc_decode_chain(mat, full)
    parts = torch.full((T * 9,), float("nan"), dtype=torch.float16, device=DEV)
    for p in range(nparts):
        ntc.ntc_decode_chain_part(mat, p, nparts, parts)
    torch.cuda.synchronize()
    assert torch.equal(full.view(torch.int16), parts.view(torch.int16))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _setup():
    import oracle as O
    from paper_2305_17105_b200.synth import (box_mip_chain_u8, gen_crops, gen_latents, gen_reference_u8,
                                             gen_weights_f32, u8_to_f16_bits)

    d = Profile.named("ntc0.2", 128, 8)
    lat = gen_latents(1, O.num_latents(d))
    par = gen_weights_f32(2, d.input_dim, 8)
    ref = u8_to_f16_bits(box_mip_chain_u8(gen_reference_u8(3, 128, 8))[0])
    gcrops = gen_crops(4, 128, 0, 5, 32)
    return d, lat, par, ref, gcrops


def _setup_chain():
    """_setup's material with the whole reference mip chain (fp16 bits per mip)."""
    from paper_2305_17105_b200.synth import box_mip_chain_u8, gen_reference_u8, u8_to_f16_bits

    d, lat, par, _, _ = _setup()
    return d, lat, par, [u8_to_f16_bits(m) for m in box_mip_chain_u8(gen_reference_u8(3, 128, 8))]


def _worker(rank, world, port, q):
    import sys

    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2305_17105_b200 as ntc
        from paper_2305_17105_b200.dist import DataParallelTrainer

        d, lat, par, ref, gcrops = _setup()
        tr = DataParallelTrainer(d, torch.from_numpy(lat).to(DEV), torch.from_numpy(par).to(DEV))
        refd = torch.from_numpy(ref.view(np.int16)).to(DEV)
        hp = ntc.Hparams(0.01, 0.005, 0.9, 0.999, 1e-8, 1, 7, 1, 0)
        loss = tr.step(0, gcrops, refd, 128 * 8, hp)
        torch.cuda.synchronize()
        q.put((rank, float(loss.item()), tr.t["grad_par"].cpu().numpy().copy(), tr.t["grad_lat"].cpu().numpy().copy(),
               tr.t["params"].cpu().numpy().copy(), tr.t["latents"].cpu().numpy().copy()))
    finally:
        dist.destroy_process_group()


def test_dp_step_two_ranks_matches_single_batch():
    """2-rank DP step == one GRADS+APPLY on the global batch: loss, all-reduced gradients
    (fp32 summation order only) and identical replicas after the Adam step."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(2)], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # single-process reference on the same GPU
    d, lat, par, ref, gcrops = _setup()
    NL, P = lat.size, par.size
    t = {k: torch.zeros(NL, device=DEV) for k in ("m_lat", "v_lat", "grad_lat", "noisy")}
    t.update({k: torch.zeros(P, device=DEV) for k in ("m_par", "v_par", "grad_par")})
    t["latents"] = torch.from_numpy(lat.copy()).to(DEV)
    t["params"] = torch.from_numpy(par.copy()).to(DEV)
    refd = torch.from_numpy(ref.view(np.int16)).to(DEV)
    loss = torch.zeros(1, device=DEV)
    ntc.ntc_train_step(ntc.Trainer(d), ntc.make_buffers(t), ntc.make_batch(0, gcrops, refd, 128 * 8),
                       ntc.Hparams(0.01, 0.005, 0.9, 0.999, 1e-8, 1, 7, 1, 0), loss, flags=ntc.NTC_STEP_GRADS)
    torch.cuda.synchronize()
    gp, gl = t["grad_par"].cpu().numpy(), t["grad_lat"].cpu().numpy()
    for r in res:
        _, l, dgp, dgl, _, _ = r
        assert abs(l - loss.item()) <= 1e-5 * loss.item()
        assert np.linalg.norm(dgp - gp) <= 1e-5 * np.linalg.norm(gp)
        assert np.linalg.norm(dgl - gl) <= 1e-5 * np.linalg.norm(gl)
    assert np.array_equal(res[0][4], res[1][4]) and np.array_equal(res[0][5], res[1][5])


def _shard_worker(rank, world, port, q, steps, mip=0, crop=32):
    import sys

    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2305_17105_b200 as ntc
        from paper_2305_17105_b200.dist import ShardedDataParallelTrainer
        from paper_2305_17105_b200.synth import gen_crops

        d, lat, par, ref = _setup_chain()
        tr = ShardedDataParallelTrainer(d, torch.from_numpy(lat).to(DEV), torch.from_numpy(par).to(DEV))
        refd = [torch.from_numpy(r.view(np.int16)).to(DEV) for r in ref]
        losses = []
        for s in range(steps):
            hp = ntc.Hparams(0.01, 0.005, 0.9, 0.999, 1e-8, s + 1, 7, 1, 0)
            crops = gen_crops(40 + s, 128, mip, 6, crop)
            losses.append(float(tr.step(mip, crops, refd[mip], (128 >> mip) * 8, hp).item()))
        full = tr.gather_latents()
        torch.cuda.synchronize()
        q.put((rank, losses, tr.t["params"].cpu().numpy().copy(), full.cpu().numpy().copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,mip,crop", [(2, 0, 32), (3, 3, 12), (3, 4, 6)])
def test_sharded_dp_matches_single_process(world, mip, crop):
    """Latent grids sharded by row bands (2-3 ranks): after 3 GRADS+APPLY steps the gathered
    latents and the weights equal single-process training on the same global batches (fp32
    summation order only), and the ranks agree.  At mips 3-4 every crop spans several bands,
    so boxes that different readers send back to one owner overlap (their halo-gradient adds
    must not race: ADVICE r1).  Latents: see the bound below."""
    from paper_2305_17105_b200.synth import gen_crops

    steps = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, world, port, q, steps, mip, crop)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    d, lat, par, ref = _setup_chain()
    NL, P = lat.size, par.size
    t = {k: torch.zeros(NL, device=DEV) for k in ("m_lat", "v_lat", "grad_lat", "noisy")}
    t.update({k: torch.zeros(P, device=DEV) for k in ("m_par", "v_par", "grad_par")})
    t["latents"] = torch.from_numpy(lat.copy()).to(DEV)
    t["params"] = torch.from_numpy(par.copy()).to(DEV)
    refd = [torch.from_numpy(r.view(np.int16)).to(DEV) for r in ref]
    tr, bufs, loss = ntc.Trainer(d), ntc.make_buffers(t), torch.zeros(1, device=DEV)
    losses = []
    for s in range(steps):
        hp = ntc.Hparams(0.01, 0.005, 0.9, 0.999, 1e-8, s + 1, 7, 1, 0)
        crops = gen_crops(40 + s, 128, mip, 6, crop)
        ntc.ntc_train_step(tr, bufs, ntc.make_batch(mip, crops, refd[mip], (128 >> mip) * 8), hp, loss)
        losses.append(float(loss.item()))
    torch.cuda.synchronize()
    ref_lat, ref_par = t["latents"].cpu().numpy(), t["params"].cpu().numpy()
    for _, l, p, full in res:
        assert np.allclose(l, losses, rtol=1e-5)
        assert np.allclose(p, ref_par, rtol=1e-4, atol=1e-6)
        # The two runs sum the same fp32 gradient contributions in different orders (ranks,
        # atomics); from step 2 on the 1-ulp weight differences can flip fp16 activation
        # roundings, and Adam normalises whatever gradient difference results.  A lost or
        # doubled halo contribution moves a latent by O(lr_latent) per step (Adam's update
        # size), reordering by ~1e-5 (measured: <= 8e-6 over 3 steps at mip 4): the bound
        # 2e-3 * lr_latent * steps separates the two by > 100x.
        atol = 2e-3 * 0.01 * steps
        assert np.abs(full - ref_lat).max() <= atol, np.abs(full - ref_lat).max()
    for r in res[1:]:
        assert np.array_equal(res[0][2], r[2]) and np.array_equal(res[0][3], r[3])


def test_bench_two_ranks_json_line():
    """bench.py's N > 1 path (torchrun, two ranks sharing cuda:0 over gloo): one JSON line
    with the contract's keys, weak-scaling totals over both ranks, and the sharded
    data-parallel training step."""
    import json
    import subprocess
    import sys

    env = dict(os.environ, NTC_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--no-extras", "--c5-materials", "4"]
    out = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    r = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "dtype", "config", "roofline", "gpu_launches", "clocks", "e2e", "train"):
        assert k in r, k
    assert r["n_gpus"] == 2 and r["scaling"] == "weak" and r["value"] > 0
    assert "sharded" in r["train"]["parallelism"]
    assert r["comm"]["world"] == 2 and r["comm"]["allreduce_of_ones"] == 2.0
    assert r["train_uniform"]["halo_latents_received_per_step_max_rank"] > 0  # R19 crops cross bands
    c5 = r["c5"]
    assert c5["materials"] == 4 and c5["decode"]["value"] > 0 and c5["train_mp"]["value"] > 0
    assert c5["train_dp"]["value"] > 0 and "stacked all-reduce" in c5["train_dp"]["parallelism"]


def _stacked_worker(rank, world, port, q, steps, mip, crop, M):
    import sys

    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2305_17105_b200 as ntc
        from paper_2305_17105_b200.dist import StackedDataParallelTrainer
        from paper_2305_17105_b200.synth import gen_crops, gen_latents, gen_weights_f32

        d, _, _, ref = _setup_chain()
        NL = ntc.ntc_num_latents(d)
        lats = [torch.from_numpy(gen_latents(100 + k, NL)).to(DEV) for k in range(M)]
        pars = [torch.from_numpy(gen_weights_f32(200 + k, d.input_dim, 8)).to(DEV) for k in range(M)]
        tr = StackedDataParallelTrainer(d, lats, pars)
        refd = torch.from_numpy(ref[mip].view(np.int16)).to(DEV)
        losses = []
        for s in range(steps):
            hp = ntc.Hparams(0.01, 0.005, 0.9, 0.999, 1e-8, s + 1, 7, 1, 0)
            crops = [gen_crops(40 + 10 * k + s, 128, mip, 6, crop) for k in range(M)]
            losses.append(tr.step(mip, crops, [refd] * M, (128 >> mip) * 8, hp).cpu().numpy().copy())
        full = [tr.gather_latents(k).cpu().numpy().copy() for k in range(M)]
        pars_out = [tr.mats[k].t["params"].cpu().numpy().copy() for k in range(M)]
        torch.cuda.synchronize()
        q.put((rank, np.array(losses), pars_out, full, tr.launches))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,mip,crop", [(2, 0, 32), (3, 3, 12)])
def test_stacked_materials_match_single_process(world, mip, crop):
    """C5's stacked data-parallel trainer (several materials, latents sharded by row bands,
    one batched halo all-to-all each way and ONE all-reduce of every material's [dW | loss])
    equals training each material alone on the same global batches."""
    from paper_2305_17105_b200.synth import gen_crops, gen_latents, gen_weights_f32

    M, steps = 3, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_stacked_worker, args=(r, world, port, q, steps, mip, crop, M))
             for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    d, _, _, ref = _setup_chain()
    NL, P = ntc.ntc_num_latents(d), ntc.ntc_num_params(d)
    refd = torch.from_numpy(ref[mip].view(np.int16)).to(DEV)
    for k in range(M):
        t = {n: torch.zeros(NL, device=DEV) for n in ("m_lat", "v_lat", "grad_lat", "noisy")}
        t.update({n: torch.zeros(P, device=DEV) for n in ("m_par", "v_par", "grad_par")})
        t["latents"] = torch.from_numpy(gen_latents(100 + k, NL)).to(DEV)
        t["params"] = torch.from_numpy(gen_weights_f32(200 + k, d.input_dim, 8)).to(DEV)
        tr, bufs, loss = ntc.Trainer(d), ntc.make_buffers(t), torch.zeros(1, device=DEV)
        losses = []
        for s in range(steps):
            hp = ntc.Hparams(0.01, 0.005, 0.9, 0.999, 1e-8, s + 1, 7, 1, 0)
            crops = gen_crops(40 + 10 * k + s, 128, mip, 6, crop)
            ntc.ntc_train_step(tr, bufs, ntc.make_batch(mip, crops, refd, (128 >> mip) * 8), hp, loss)
            losses.append(float(loss.item()))
        torch.cuda.synchronize()
        for _, l, p, full, _ in res:
            assert np.allclose(l[:, k], losses, rtol=1e-5)
            assert np.allclose(p[k], t["params"].cpu().numpy(), rtol=1e-4, atol=1e-6)
            # latent bound: see test_sharded_dp_matches_single_process
            assert np.abs(full[k] - t["latents"].cpu().numpy()).max() <= 2e-3 * 0.01 * steps


def _nccl_worker(q, steps, mip, crop):
    """One rank over NCCL (a real NCCL communicator on cuda:0; two ranks cannot share one GPU
    under NCCL): the device-side collectives of the sharded and stacked trainers run."""
    import sys

    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        import paper_2305_17105_b200 as ntc
        from paper_2305_17105_b200.dist import ShardedDataParallelTrainer, StackedDataParallelTrainer
        from paper_2305_17105_b200.synth import gen_crops

        assert dist.get_backend() == "nccl"
        d, lat, par, ref = _setup_chain()
        refd = torch.from_numpy(ref[mip].view(np.int16)).to(DEV)
        sh = ShardedDataParallelTrainer(d, torch.from_numpy(lat.copy()).to(DEV), torch.from_numpy(par.copy()).to(DEV))
        st = StackedDataParallelTrainer(d, [torch.from_numpy(lat.copy()).to(DEV)], [torch.from_numpy(par.copy()).to(DEV)])
        out = []
        for s in range(steps):
            hp = ntc.Hparams(0.01, 0.005, 0.9, 0.999, 1e-8, s + 1, 7, 1, 0)
            crops = gen_crops(40 + s, 128, mip, 6, crop)
            l1 = float(sh.step(mip, crops, refd, (128 >> mip) * 8, hp).item())
            l2 = float(st.step(mip, [crops], [refd], (128 >> mip) * 8, hp)[0].item())
            out.append((l1, l2))
        g = sh.gather_latents()  # the NCCL all-to-all of the band exchange
        torch.cuda.synchronize()
        q.put((out, sh.t["params"].cpu().numpy(), st.mats[0].t["params"].cpu().numpy(), g.cpu().numpy(),
               sh.t["latents"].cpu().numpy()))
    finally:
        dist.destroy_process_group()


def test_nccl_single_rank_trainers():
    """The NCCL code paths of dist.py (device all-reduce, all-to-all) on a one-rank NCCL group:
    the sharded and the stacked trainer agree with each other and with single-process training
    of the same batches (a one-rank all-reduce is the identity)."""
    from paper_2305_17105_b200.synth import gen_crops

    steps, mip, crop = 2, 1, 24
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_worker, args=(q, steps, mip, crop))
    p.start()
    out, p_sh, p_st, gathered, lat_sh = q.get(timeout=300)
    p.join(timeout=60)
    assert p.exitcode == 0
    d, lat, par, ref = _setup_chain()
    NL, P = lat.size, par.size
    t = {k: torch.zeros(NL, device=DEV) for k in ("m_lat", "v_lat", "grad_lat", "noisy")}
    t.update({k: torch.zeros(P, device=DEV) for k in ("m_par", "v_par", "grad_par")})
    t["latents"] = torch.from_numpy(lat.copy()).to(DEV)
    t["params"] = torch.from_numpy(par.copy()).to(DEV)
    refd = torch.from_numpy(ref[mip].view(np.int16)).to(DEV)
    tr, bufs, loss = ntc.Trainer(d), ntc.make_buffers(t), torch.zeros(1, device=DEV)
    for s in range(steps):
        hp = ntc.Hparams(0.01, 0.005, 0.9, 0.999, 1e-8, s + 1, 7, 1, 0)
        ntc.ntc_train_step(tr, bufs, ntc.make_batch(mip, gen_crops(40 + s, 128, mip, 6, crop), refd, (128 >> mip) * 8),
                           hp, loss)
        assert abs(out[s][0] - float(loss.item())) <= 1e-5 * abs(float(loss.item()))
        assert abs(out[s][1] - float(loss.item())) <= 1e-5 * abs(float(loss.item()))
    torch.cuda.synchronize()
    assert np.allclose(p_sh, t["params"].cpu().numpy(), rtol=1e-4, atol=1e-6)
    assert np.allclose(p_st, p_sh, rtol=1e-4, atol=1e-6)
    assert np.array_equal(gathered, lat_sh)  # one rank: the gathered bands are its own latents
    assert np.abs(lat_sh - t["latents"].cpu().numpy()).max() <= 2e-3 * 0.01 * steps
