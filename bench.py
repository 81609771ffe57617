#!/usr/bin/env python
"""NTC hot-path benchmark (BASELINE.json metric: decoded Gtexel/s on the 4K 9-channel
full mip chain, and training texels/s).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one pass of the hot path over synthetic inputs resident in HBM:
  decode  : ntc_decode_chain of a 4096^2, 9-channel, NTC 0.2 material (22,369,621 texels)
  train   : ntc_train_step(GRADS|APPLY) on 4 random 256^2 crops at LOD 0 (262,144 texels)
            of a 4096^2 9-channel material (configs[3]), when the library provides it.
L2 is flushed (256 MiB write) before every timed step, outside the CUDA-event window.
Extra lines at N=1 (--no-extras skips them): `random` = configs[2]'s 2^24 random-access
queries on a 4096^2 16-channel material; `multi` = the Table 4 screen workload over 8 materials
(f3); `configs` = the other SURVEY.md 8(d) rows (C1, C2, C3a, stress, C4 LOD mix, variants).
`c5` at every N (--no-c5 skips it): configs[4], 64 materials -- material-parallel decode and
training, and at N > 1 the stacked data-parallel trainer (one all-reduce for all materials).
Multi-GPU (torchrun): weak scaling, one independent material per rank for the headline decode
(no collective), the sharded data-parallel training step (stratified crops, plus a
`train_uniform` line with the R19 placement whose halos cross bands) and a `comm` record (backend,
NCCL version, all-reduce of ones = rank count); time = max over ranks of the device time.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2305_17105_b200.synth import (SEED_BASE, Profile, box_mip_chain_u8, gen_codes, gen_crops,  # noqa: E402
                                         gen_latents, gen_queries, gen_reference_u8, gen_weights_f16,
                                         gen_weights_f32, u8_to_f16_bits)

METRIC = "decoded Gtexel/s (4K 9-ch material, full mip chain) and training texels/s"
UNIT = "Gtexel/s"
W, C = 4096, 9
WORKLOAD = "4096^2 x 9ch NTC0.2 [57,64,64,9] full-chain decode (22,369,621 texels)"
TRAIN_WORKLOAD = "4096^2 x 9ch NTC0.2 train step, 4 x 256^2 crops at LOD 0 (262,144 texels)"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return pk, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


def _ncu_metric(kernel, name):
    """One metric value of `kernel` in the committed ncu summary (or None)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            return float(json.load(f)["kernels"][kernel]["metrics"][name][0])
    except Exception:
        return None


def _ncu_instructions(kernel):
    """warp instructions per launch of `kernel` from the committed ncu summary (or None)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            return float(json.load(f)["kernels"][kernel]["instructions_per_launch"])
    except Exception:
        return None


def _issue_ceiling(torch, dev, instr_per_launch, units, sm_mhz):
    """The instruction-issue roofline of a kernel: every SM sub-partition issuing one warp
    instruction per cycle (4 per SM) at the sampled SM clock, divided by the kernel's warp
    instructions per unit (ncu).  Returns (units/s ceiling, thread instructions per unit)."""
    if not instr_per_launch or not sm_mhz:
        return None, None
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    per_unit = instr_per_launch / units
    return 4 * sms * sm_mhz * 1e6 / per_unit, 32 * per_unit


def _ncu_traffic(kernel):
    """dram read+write bytes per launch of `kernel` from the committed ncu summary (or None)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            s = json.load(f)
        return s["kernels"][kernel]["dram_bytes_per_launch"]
    except Exception:
        return None


class ClockSampler:
    """NVML sampling of SM clocks and clock-event (throttle) reasons during the timed region."""

    NAMES = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
             0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
             0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index):
        self.samples, self.reasons, self.ok = [], 0, False
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def report(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max, "reasons": ["unavailable"]}
        rs = [n for b, n in self.NAMES.items() if self.reasons & b and n != "gpu_idle"]
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max, "reasons": rs,
                "samples": len(self.samples)}


def decode_flops_per_texel(d):
    """Unpadded algorithmic FLOPs per decoded texel: 2 (D*64 + 4096 h + 64 c)."""
    return 2 * (d.input_dim * 64 + 4096 * d.hidden_mats + 64 * d.channels)


def train_flops_per_texel(d):
    """forward + dX (hidden, latent inputs) + dW."""
    h = d.hidden_mats
    fwd = d.input_dim * 64 + 4096 * h + 64 * d.channels
    bwd = 64 * d.channels + 4096 * h + (4 * d.c0 + d.c1) * 64 + 64 * d.channels + 4096 * h + 64 * d.input_dim
    return 2 * (fwd + bwd)


# ------------------------------------------------------------------------------------ ours
def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_2305_17105_b200 as ntc

    dev = torch.device("cuda", local_rank % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    stream = torch.cuda.current_stream()
    d = Profile.named("ntc0.2", W, C)
    seed = SEED_BASE + 4 + rank  # configs[4]: per-material seed = base + material id
    codes = gen_codes(seed, ntc.grid_list(d))
    wts = gen_weights_f16(seed + 1, d.input_dim, C)
    codes_d = torch.from_numpy(codes).to(dev)
    w_d = torch.from_numpy(wts.view(np.int16)).to(dev)
    mat = ntc.Material(d, codes_d, w_d)
    T = ntc.ntc_chain_texels(d)
    out = torch.empty((T * C,), dtype=torch.float16, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    # training state (configs[3]) if the library provides the step
    train = None
    try:
        tr = ntc.Trainer(d)
        NL, P = ntc.ntc_num_latents(d), ntc.ntc_num_params(d)
        tb = {k: torch.zeros(NL, device=dev) for k in ("m_lat", "v_lat", "grad_lat", "noisy")}
        tb.update({k: torch.zeros(P, device=dev) for k in ("m_par", "v_par", "grad_par")})
        tb["latents"] = torch.from_numpy(gen_latents(seed + 2, NL)).to(dev)
        tb["params"] = torch.from_numpy(gen_weights_f32(seed + 3, d.input_dim, C)).to(dev)
        ref0 = torch.from_numpy(u8_to_f16_bits(gen_reference_u8(seed + 4, W, C)).view(np.int16)).to(dev)
        train = dict(tr=tr, tb=tb, buf=ntc.make_buffers(tb), ref=ref0, loss=torch.zeros(1, device=dev),
                     status=torch.zeros(1, dtype=torch.int32, device=dev))
    except ntc.NtcError as e:
        if e.status != ntc.NTC_ERR_UNSUPPORTED:
            raise

    # weak scaling: 4 crops of 256^2 per rank; all ranks draw the same global crop list.  At
    # N > 1 the latent grids are sharded by row bands (ShardedDataParallelTrainer) and the 4
    # crops of each rank are drawn inside its band (stratified placement, balanced owners).
    dp = None
    if train is not None and world > 1:
        from paper_2305_17105_b200.dist import ShardedDataParallelTrainer, stratified_crops

        dp = ShardedDataParallelTrainer(d, train["tb"]["latents"], train["tb"]["params"])
        crop_sets = [stratified_crops(d, 0, world, 4, 256, np.random.default_rng(SEED_BASE + 3 + 1000 * i))
                     for i in range(args.warmup + args.steps)]
        # the host-side step schedules (crop ownership, halo boxes) are built ahead of the loop,
        # as a training loop builds them a step early from the seeded crop list
        plans = [dp.plan(0, c) for c in crop_sets]
    else:
        crop_sets = [gen_crops(SEED_BASE + 3 + 1000 * i, W, 0, 4, 256) for i in range(args.warmup + args.steps)]
    launches = {"train": 0}

    def train_step(i):
        hp = ntc.Hparams(0.01, 0.005, 0.9, 0.999, 1e-8, i + 1, seed, 1, 0)
        if dp is not None:  # sharded data-parallel: halo all-to-all, GRADS, grad all-to-all, all-reduce, APPLY
            dp.step(0, crop_sets[i], train["ref"], W * C, hp, plan=plans[i])
            launches["train"] += dp.launches
            return
        batch = ntc.make_batch(0, crop_sets[i], train["ref"], W * C)
        ntc.ntc_train_step(train["tr"], train["buf"], batch, hp, train["loss"], train["status"])
        launches["train"] += 3  # prep (+ weight image), fused forward/backward, reduce + Adam

    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]

    def step(i, timed):
        flush.zero_()
        ev[0].record(stream)
        ntc.ntc_decode_chain(mat, out)
        ev[1].record(stream)
        if train is not None:
            train_step(i)
        ev[2].record(stream)
        if timed:
            ev[2].synchronize()
            return (ev[0].elapsed_time(ev[2]) / 1e3, ev[0].elapsed_time(ev[1]) / 1e3,
                    ev[1].elapsed_time(ev[2]) / 1e3)
        return None

    for i in range(args.warmup):
        step(i, False)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    tot = dec = trn = 0.0
    launches["train"] = 0
    with ClockSampler(local_rank) as clk:
        for i in range(args.steps):
            a, b, c = step(args.warmup + i, True)
            tot += a
            dec += b
            trn += c
    torch.cuda.synchronize()
    if world > 1:
        t = torch.tensor([tot, dec, trn], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.barrier()
        tot, dec, trn = t.tolist()

    texels = T * world * args.steps
    res = {}
    pk, pk_src = _peaks()
    peak_tf = pk["bf16_tflops"]
    dec_flops = decode_flops_per_texel(d) * T
    achieved = dec_flops / (dec / args.steps) / 1e12
    tr_bytes = _ncu_traffic("decode")
    res.update({
        "metric": METRIC, "value": texels / dec / 1e9, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": tot / args.steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f16 (fp32 accumulate)",
        "data": "synthetic (seeded iid codes, He-uniform fp16 weights; DESIGN.md input recipe)",
        "config": {"workload": WORKLOAD, "profile": "ntc0.2", "width": W, "channels": C,
                   "texels_per_step_per_gpu": T, "l2": "flushed (256 MiB write) before each timed step",
                   "parallelism": f"material-parallel x{world} (no collective)"},
        "roofline": {"bound": "tensor", "achieved": round(achieved, 2), "peak": peak_tf, "unit": "TFLOP/s",
                     "frac": round(achieved / peak_tf, 4), "traffic": tr_bytes,
                     "peak_source": f"{pk_src} bf16 dense burst (fp16 same rate)",
                     "kernel": "ntc::decode_kernel", "flops_per_texel": decode_flops_per_texel(d),
                     # SURVEY 8(d) diagnostics: HBM use of the same launch (live time, committed ncu
                     # bytes) and the issue-slot utilisation that bounds the kernel (ncu)
                     "diagnostics": {
                         "dram_gbs": None if tr_bytes is None else round(tr_bytes / (dec / args.steps) / 1e9, 1),
                         "dram_frac": None if tr_bytes is None else
                         round(tr_bytes / (dec / args.steps) / 1e9 / pk["hbm_gbs"], 4),
                         "issue_active_pct": _ncu_metric("decode", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
                         "tensor_pipe_pct": _ncu_metric(
                             "decode", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active")}},
        "gpu_launches": args.steps + launches["train"],
        "clocks": clk.report(),
    })
    # the bound that actually binds the decode: instruction issue on the ALU work
    # around the contractions -- the texel rate at one warp instruction per sub-partition per
    # cycle, and the fraction of it reached (diagnostic; `frac` above stays the tensor roofline)
    ceil_t, ipt = _issue_ceiling(torch, dev, _ncu_instructions("decode"), T,
                                 res["clocks"].get("sm_mhz") or res["clocks"].get("sm_max_mhz"))
    if ceil_t:
        res["roofline"]["diagnostics"].update({
            "thread_instructions_per_texel": round(ipt, 1),
            "issue_ceiling_gtexel_s": round(ceil_t / 1e9, 2),
            "frac_of_issue_ceiling": round(res["value"] / (ceil_t / 1e9 * world), 4)})
    if train is not None:
        B = 4 * 256 * 256
        tflops = train_flops_per_texel(d) * B / (trn / args.steps) / 1e12
        res["train"] = {"metric": "training texels/s", "value": B * world * args.steps / trn,
                        "parallelism": "single GPU" if world == 1 else
                        f"data-parallel x{world}, latent grids sharded by row bands: 4 crops/rank inside its band, "
                        "NCCL all-to-all of halo latents and halo gradients, all-reduce of [dW | loss]",
                        "unit": "texel/s", "ms_per_step": trn / args.steps * 1e3, "workload": TRAIN_WORKLOAD,
                        "roofline": {"bound": "tensor", "achieved": round(tflops, 2), "peak": peak_tf,
                                     "unit": "TFLOP/s", "frac": round(tflops / peak_tf, 4),
                                     "kernel": "ntc::train_kernel (+ prep, reduce/Adam in the step time)",
                                     "flops_per_texel": train_flops_per_texel(d),
                                     "diagnostics": {
                                         "issue_active_pct": _ncu_metric(
                                             "train", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
                                         "tensor_pipe_pct": _ncu_metric(
                                             "train", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active")}}}
    # e2e through the public API from pinned host buffers (rank 0 and every rank alike)
    res["e2e"] = e2e(args, ntc, torch, d, codes, wts, dev, world)
    if world > 1:
        res["comm"] = comm_check(torch, dist, dev, world)
        if train is not None:
            res["train_uniform"] = bench_train_uniform(args, ntc, torch, dev, flush, d, train, world)
    if not args.no_c5:
        res["c5"] = bench_c5(args, ntc, torch, dev, flush, rank, world)
    if world == 1 and not args.no_extras:
        res["random"] = bench_random(args, ntc, torch, dev, flush)
        res["multi"] = bench_multi(args, ntc, torch, dev, flush)
        res["configs"] = bench_configs(args, ntc, torch, dev, flush)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        res["cpu_baseline"] = cpu_baseline(d, codes, wts, budget_s=args.cpu_budget)
    return res


def _device_time(torch, fn, flush, reps):
    """mean device seconds of fn() over `reps` runs, L2 flushed before each (outside the events)"""
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    tot = 0.0
    for _ in range(reps):
        flush.zero_()
        e0.record(s)
        fn()
        e1.record(s)
        e1.synchronize()
        tot += e0.elapsed_time(e1) / 1e3
    return tot / reps


def bench_random(args, ntc, torch, dev, flush):
    """configs[2] (C3b): 2^24 random-access queries, area-uniform over the chain, random order,
    on a 4096^2 16-channel NTC 0.2 material (ntc_decode_texels)."""
    d = Profile.named("ntc0.2", W, 16)
    seed = SEED_BASE + 2
    mat = ntc.Material(d, torch.from_numpy(gen_codes(seed, ntc.grid_list(d))).to(dev),
                       torch.from_numpy(gen_weights_f16(seed + 1, d.input_dim, 16).view(np.int16)).to(dev))
    n = 1 << 24
    q = ntc.pack_queries(torch.from_numpy(gen_queries(seed + 2, W, n, "area")).to(dev))
    out = torch.empty((n, 16), dtype=torch.float16, device=dev)
    t = _device_time(torch, lambda: ntc.ntc_decode_texels(mat, q, out), flush, max(3, min(args.steps, 10)))
    pk, _ = _peaks()
    tf = decode_flops_per_texel(d) * n / t / 1e12
    return {"metric": "random-access decoded Gtexel/s", "value": n / t / 1e9, "unit": UNIT,
            "workload": "4096^2 x 16ch NTC0.2, 2^24 area-uniform random queries (configs[2])",
            "ms_per_step": t * 1e3, "roofline": {"bound": "tensor", "achieved": round(tf, 2),
                                                 "peak": pk["bf16_tflops"], "unit": "TFLOP/s",
                                                 "frac": round(tf / pk["bf16_tflops"], 4)}}


def _material(ntc, torch, d, seed, dev, out_gain=0.3):
    return ntc.Material(d, torch.from_numpy(gen_codes(seed, ntc.grid_list(d))).to(dev),
                        torch.from_numpy(gen_weights_f16(seed + 1, d.input_dim, d.channels, d.hidden_mats,
                                                         out_gain=out_gain).view(np.int16)).to(dev))


def _row(d, texels, t, flops_per_texel, peak, **kw):
    tf = flops_per_texel * texels / t / 1e12
    r = {"texels": int(texels), "ms": round(t * 1e3, 4), "Gtexel_s": round(texels / t / 1e9, 3),
         "tflops": round(tf, 1), "frac": round(tf / peak, 4)}
    r.update(kw)
    return r


VARIANTS = [("ntc0.5", 1, 0), ("ntc1.0", 1, 0), ("ntc2.25", 1, 0), ("ntc0.2", 2, 0), ("ntc0.2", 1, 1)]


def bench_configs(args, ntc, torch, dev, flush):
    """The other SURVEY.md 8(d) rows, each timed like the headline (L2 flushed before every
    run, CUDA events on the launching stream, mean of `reps`), with its tensor-roofline
    fraction (unpadded algorithmic FLOPs / measured burst peak):
      C1  configs[0]: 256^2 x 8ch, mip 0 only (65,536 texels, one ntc_decode_mip)
      C2  configs[1]: 2048^2 x 9ch full chain (5,592,405 texels)
      C3a configs[2]: 4096^2 x 16ch full chain (22,369,621 texels)
      stress: the headline material with output-layer gain 1.0 (many clamped outputs)
      C4_lod_mix configs[3]: training steps whose LOD follows the paper's law
      variants: the other Table 2 profiles, depth reading B and exact GELU, decode and train."""
    pk, _ = _peaks()
    peak = pk["bf16_tflops"]
    reps = max(3, min(args.steps, 10))
    res = {}

    def chain(name, d, seed, gain=0.3, **kw):
        mat = _material(ntc, torch, d, seed, dev, gain)
        T = ntc.ntc_chain_texels(d)
        out = torch.empty((T * d.channels,), dtype=torch.float16, device=dev)
        t = _device_time(torch, lambda: ntc.ntc_decode_chain(mat, out), flush, reps)
        return _row(d, T, t, decode_flops_per_texel(d), peak, **kw)

    d1 = Profile.named("ntc0.2", 256, 8)
    m1 = _material(ntc, torch, d1, SEED_BASE + 0, dev)
    o1 = torch.empty((256 * 256 * 8,), dtype=torch.float16, device=dev)
    t1 = _device_time(torch, lambda: ntc.ntc_decode_mip(m1, 0, o1), flush, reps)
    res["C1"] = _row(d1, 256 * 256, t1, decode_flops_per_texel(d1), peak,
                     workload="256^2 x 8ch NTC0.2, mip 0 (configs[0]); one launch, launch-latency bound",
                     launches=1)
    res["C2"] = chain("C2", Profile.named("ntc0.2", 2048, 9), SEED_BASE + 1,
                      workload="2048^2 x 9ch NTC0.2 full chain (configs[1])")
    res["C3a"] = chain("C3a", Profile.named("ntc0.2", W, 16), SEED_BASE + 2,
                       workload="4096^2 x 16ch NTC0.2 full chain (configs[2])")
    res["stress"] = chain("stress", Profile.named("ntc0.2", W, C), SEED_BASE + 4, gain=1.0,
                          workload="4096^2 x 9ch NTC0.2 full chain, stress weights (output gain 1.0)")
    res["variants_decode"] = [
        chain(name, Profile.named(name, W, C, hm, act), SEED_BASE + 4, profile=name, hidden_mats=hm,
              activation=["hardGELU", "GELU"][act])
        for name, hm, act in VARIANTS]

    # training: LOD mix (configs[3]) and the variants at LOD 0
    ref_chain = [torch.from_numpy(u8_to_f16_bits(m).view(np.int16)).to(dev)
                 for m in box_mip_chain_u8(gen_reference_u8(SEED_BASE + 8, W, C))]

    def trainer(d, seed):
        NL, P = ntc.ntc_num_latents(d), ntc.ntc_num_params(d)
        t = {k: torch.zeros(NL, device=dev) for k in ("m_lat", "v_lat", "grad_lat", "noisy")}
        t.update({k: torch.zeros(P, device=dev) for k in ("m_par", "v_par", "grad_par")})
        t["latents"] = torch.from_numpy(gen_latents(seed, NL)).to(dev)
        t["params"] = torch.from_numpy(gen_weights_f32(seed + 1, d.input_dim, d.channels, d.hidden_mats)).to(dev)
        return ntc.Trainer(d), t, ntc.make_buffers(t), torch.zeros(1, device=dev)

    def train_time(d, batches, seed):
        tr, t, bufs, loss = trainer(d, seed)
        step = [0]

        def run_all():
            for b in batches:
                step[0] += 1
                ntc.ntc_train_step(tr, bufs, b, ntc.Hparams(0.01, 0.005, 0.9, 0.999, 1e-8, step[0], 7, 1, 0), loss)

        return _device_time(torch, run_all, flush, reps)

    from paper_2305_17105_b200.compress import sample_lod

    d = Profile.named("ntc0.2", W, C)
    M = ntc.ntc_num_mips(d)
    rng = np.random.default_rng(SEED_BASE + 9)
    batches, texels, lods = [], 0, []
    for _ in range(32):
        m = sample_lod(rng, M)
        crops = gen_crops(int(rng.integers(1 << 30)), W, m, 4, 256)
        texels += int((crops[:, 2] * crops[:, 3]).sum())
        lods.append(m)
        batches.append(ntc.make_batch(m, crops, ref_chain[m], (W >> m) * C))
    tt = train_time(d, batches, SEED_BASE + 10)
    res["C4_lod_mix"] = _row(d, texels, tt, train_flops_per_texel(d), peak,
                             workload="4096^2 x 9ch NTC0.2 train steps (GRADS|APPLY), 32 steps of 4 x 256^2 crops "
                                      "(capped at the mip size) at LODs from the paper's law (PAPER.md:572-574)",
                             steps=32, lods=lods, unit_note="Gtexel_s = G texels/s over the 32 steps")
    crops0 = gen_crops(SEED_BASE + 3, W, 0, 4, 256)
    rows = []
    for name, hm, act in [("ntc0.2", 1, 0)] + VARIANTS:
        dv = Profile.named(name, W, C, hm, act)
        b = [ntc.make_batch(0, crops0, ref_chain[0], W * C)]
        rows.append(_row(dv, 4 * 256 * 256, train_time(dv, b, SEED_BASE + 11), train_flops_per_texel(dv), peak,
                         profile=name, hidden_mats=hm, activation=["hardGELU", "GELU"][act]))
    res["variants_train"] = rows
    return res


def _device_codes(ntc, torch, d, seed, dev):
    """iid uniform codes of every grid (the synth.gen_codes recipe), drawn on the device from
    a seeded generator: 64 materials x 12.3 M codes are set up in milliseconds."""
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    parts = [torch.randint(0, 1 << b, (n,), generator=g, device=dev, dtype=torch.uint8)
             for n, b in ntc.grid_list(d)]
    return torch.cat(parts)


def _device_latents(ntc, torch, d, seed, dev):
    """U(-0.2, 0.2) fp32 training latents (the synth.gen_latents recipe), seeded, on the device."""
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    return torch.rand(ntc.ntc_num_latents(d), generator=g, device=dev) * 0.4 - 0.2


def comm_check(torch, dist, dev, world):
    """The process group the N > 1 numbers ran on: backend, NCCL version, and an all-reduce of
    ones that must sum to the world size (the rank count, measured)."""
    t = torch.ones(1, device=dev)
    dist.all_reduce(t)
    out = {"backend": dist.get_backend(), "world": world, "allreduce_of_ones": float(t.item())}
    try:
        v = torch.cuda.nccl.version()
        out["nccl_version"] = ".".join(str(x) for x in v) if isinstance(v, tuple) else str(v)
    except Exception:
        out["nccl_version"] = None
    return out


def bench_train_uniform(args, ntc, torch, dev, flush, d, train, world):
    """The sharded data-parallel step on the compression workload's own batches: per step a
    LOD from the paper's law (R26) and 4 x N crops of min(256, w_m)^2 placed
    uniformly over that mip (R19), each owned by the rank whose band holds its origin -- crops
    straddle bands (always at the coarser mips), so the halo all-to-alls carry latents and
    gradients (the main N > 1 line draws LOD-0 crops inside each band, stratified)."""
    import torch.distributed as dist

    from paper_2305_17105_b200.compress import sample_lod
    from paper_2305_17105_b200.dist import ShardedDataParallelTrainer

    dp = ShardedDataParallelTrainer(d, train["tb"]["latents"], train["tb"]["params"])
    M = ntc.ntc_num_mips(d)
    chain = [train["ref"].view(torch.float16).reshape(W, W, C)]  # box-filtered fp16 mips
    while chain[-1].shape[0] > 1:
        a = chain[-1].float()
        chain.append((0.25 * (a[0::2, 0::2] + a[1::2, 0::2] + a[0::2, 1::2] + a[1::2, 1::2])).half())
    chain = [c.reshape(-1).view(torch.int16) for c in chain]
    reps = max(3, min(args.steps, 10))
    rng = np.random.default_rng(SEED_BASE + 91)
    steps = []
    for i in range(reps + 1):
        m = sample_lod(rng, M)
        crops = gen_crops(SEED_BASE + 90 + i, W, m, 4 * world, 256)
        steps.append((m, crops, dp.plan(m, crops)))
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    tot, halo, texels = 0.0, 0, 0
    for i, (m, crops, plan) in enumerate(steps):
        flush.zero_()
        dist.barrier()
        e0.record(s)
        dp.step(m, crops, chain[m], (W >> m) * C, ntc.Hparams(0.01, 0.005, 0.9, 0.999, 1e-8, i + 1, 7, 1, 0),
                plan=plan)
        e1.record(s)
        e1.synchronize()
        if i > 0:
            tot += e0.elapsed_time(e1) / 1e3
            halo += sum(plan.recv_sizes)
            texels += int((crops[:, 2] * crops[:, 3]).sum())
    t = torch.tensor([tot, float(halo)], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return {"value": texels / float(t[0].item()), "unit": "texel/s", "ms_per_step": float(t[0].item()) / reps * 1e3,
            "parallelism": f"data-parallel x{world}, latents sharded by row bands; per step a LOD from the paper's "
                           "law and 4 x N crops uniform over that mip (R19, R26), owner-assigned: halo all-to-alls of "
                           "latents and gradients",
            "lods": [m for m, _, _ in steps[1:]], "halo_latents_received_per_step_max_rank": int(t[1].item()) // reps}


def _device_reference_f16(torch, seed, width, channels, dev):
    """synth.gen_reference_u8's recipe (rank-3 mix of 3 smooth fields + 10% noise, unorm8) on
    the device, then R = fp16(v / 255) (R24): the field parameters come from the same seeded
    numpy stream, the per-texel noise from a seeded device generator."""
    rng = np.random.default_rng(seed)
    y = torch.arange(width, device=dev, dtype=torch.float32)[:, None] / width
    x = torch.arange(width, device=dev, dtype=torch.float32)[None, :] / width
    fields = []
    for _ in range(3):
        f = torch.zeros((width, width), device=dev)
        for o in range(4):
            fr = 2.0 ** (o + 1)
            for _ in range(2):
                a = rng.uniform(0, 2 * np.pi, 4).astype(np.float32)
                k = rng.uniform(0.5, 1.5, 2).astype(np.float32) * fr
                f += (torch.sin(2 * np.pi * float(k[0]) * x + float(a[0])) *
                      torch.cos(2 * np.pi * float(k[1]) * y + float(a[1]))) / (o + 1)
        f -= f.min()
        f /= max(float(f.max()), 1e-6)
        fields.append(f)
    mix = rng.uniform(0.0, 1.0, size=(3, channels)).astype(np.float32)
    mix /= mix.sum(0, keepdims=True)
    img = torch.stack(fields, -1) @ torch.from_numpy(mix).to(dev)
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    img = 0.9 * img + 0.1 * torch.rand(img.shape, generator=g, device=dev)
    u8 = torch.clamp(torch.round(img * 255.0), 0, 255)
    return (u8.double() / 255.0).half().view(torch.int16).reshape(-1)


def bench_c5(args, ntc, torch, dev, flush, rank, world):
    """configs[4] (C5): 64 materials of 4096^2 x 9ch NTC 0.2 (per-material seed = base +
    material id), SURVEY.md 8(e):
      decode   material-parallel: rank r decodes the full chains of materials r, r+N, ...
               (no collective) into a ring of two output buffers;
      train_mp material-parallel training: one GRADS|APPLY step (4 x 256^2 crops at LOD 0) of
               each of the rank's materials, no collective;
      train_dp (N > 1) data-parallel over texel batches of all 64 materials at once: latents
               sharded by row bands per material, one batched halo all-to-all each way and ONE
               all-reduce of the stacked [dW | loss] of the 64 materials (2.2 MB) per step.
    Every number: texels of all ranks / max over ranks of the device time (weak scaling)."""
    import torch.distributed as dist

    M = args.c5_materials
    d = Profile.named("ntc0.2", W, C)
    T = ntc.ntc_chain_texels(d)
    mine = list(range(rank, M, world))
    reps = max(3, min(args.steps, 5))
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def timed(fn):
        fn()  # warm-up
        tot = 0.0
        for _ in range(reps):
            flush.zero_()
            if world > 1:
                dist.barrier()
            e0.record(s)
            fn()
            e1.record(s)
            e1.synchronize()
            tot += e0.elapsed_time(e1) / 1e3
        t = tot / reps
        if world > 1:
            tt = torch.tensor([t], device=dev, dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t = float(tt.item())
        return t

    pk, _ = _peaks()
    peak = pk["bf16_tflops"]
    res = {"workload": f"configs[4]: {M} materials of 4096^2 x 9ch NTC0.2", "materials": M, "n_gpus": world}
    # decode: the rank's share of full chains
    mats = [ntc.Material(d, _device_codes(ntc, torch, d, SEED_BASE + 4 + k, dev),
                         torch.from_numpy(gen_weights_f16(SEED_BASE + 5 + k, d.input_dim, C).view(np.int16)).to(dev))
            for k in mine]
    ring = [torch.empty((T * C,), dtype=torch.float16, device=dev) for _ in range(2)]

    def decode_all():
        for i, m in enumerate(mats):
            ntc.ntc_decode_chain(m, ring[i & 1])

    t = timed(decode_all)
    tf = decode_flops_per_texel(d) * T * len(mine) / t / 1e12
    res["decode"] = {"value": M * T / t / 1e9, "unit": UNIT, "ms_per_step": t * 1e3,
                     "parallelism": f"material-parallel x{world}: {len(mine)} chains per rank, no collective",
                     "roofline": {"bound": "tensor", "achieved": round(tf, 2), "peak": peak, "unit": "TFLOP/s",
                                  "frac": round(tf / peak, 4)}}
    del mats, ring
    # training state for the rank's materials (material-parallel)
    refs = {}  # material k's synthetic reference (mip 0), generated on the device

    def ref(k):
        if k not in refs:
            refs[k] = _device_reference_f16(torch, SEED_BASE + 60 + k, W, C, dev)
        return refs[k]

    def state(k):
        NL, P = ntc.ntc_num_latents(d), ntc.ntc_num_params(d)
        tb = {n: torch.zeros(NL, device=dev) for n in ("m_lat", "v_lat", "grad_lat", "noisy")}
        tb.update({n: torch.zeros(P, device=dev) for n in ("m_par", "v_par", "grad_par")})
        tb["latents"] = _device_latents(ntc, torch, d, SEED_BASE + 6 + k, dev)
        tb["params"] = torch.from_numpy(gen_weights_f32(SEED_BASE + 7 + k, d.input_dim, C)).to(dev)
        return tb

    B = 4 * 256 * 256
    sts = [(k, state(k)) for k in mine]
    for k in (range(M) if world > 1 else mine):
        ref(k)
    tr = ntc.Trainer(d)
    bufs = [ntc.make_buffers(tb) for _, tb in sts]
    loss = torch.zeros(1, device=dev)
    crops = [[gen_crops(SEED_BASE + 3 + 1000 * i + k, W, 0, 4, 256) for k in range(M)] for i in range(reps + 1)]
    it = [0]

    def train_mp():
        i = it[0] % len(crops)
        it[0] += 1
        for (k, _), b in zip(sts, bufs):
            ntc.ntc_train_step(tr, b, ntc.make_batch(0, crops[i][k], ref(k), W * C),
                               ntc.Hparams(0.01, 0.005, 0.9, 0.999, 1e-8, it[0], SEED_BASE + k, 1, 0), loss)

    t = timed(train_mp)
    tf = train_flops_per_texel(d) * B * len(mine) / t / 1e12
    res["train_mp"] = {"value": M * B / t, "unit": "texel/s", "ms_per_step": t * 1e3,
                       "parallelism": f"material-parallel x{world}: {len(mine)} materials per rank, no collective",
                       "workload": f"one GRADS|APPLY step per material, 4 x 256^2 crops at LOD 0 ({M * B} texels)",
                       "roofline": {"bound": "tensor", "achieved": round(tf, 2), "peak": peak, "unit": "TFLOP/s",
                                    "frac": round(tf / peak, 4)}}
    del sts, bufs
    if world > 1:
        from paper_2305_17105_b200.dist import StackedDataParallelTrainer, stratified_crops

        all_st = [state(k) for k in range(M)]
        dp = StackedDataParallelTrainer(d, [tb["latents"] for tb in all_st], [tb["params"] for tb in all_st])
        rng = np.random.default_rng(SEED_BASE + 77)
        dcrops = [[stratified_crops(d, 0, world, 4, 256, rng) for _ in range(M)] for _ in range(reps + 1)]
        plans = [dp.plan(0, c) for c in dcrops]
        j = [0]

        def train_dp():
            i = j[0] % len(dcrops)
            j[0] += 1
            dp.step(0, dcrops[i], [ref(k) for k in range(M)], W * C,
                    ntc.Hparams(0.01, 0.005, 0.9, 0.999, 1e-8, j[0], SEED_BASE, 1, 0), plan=plans[i])

        t = timed(train_dp)
        res["train_dp"] = {"value": M * B * world / t, "unit": "texel/s", "ms_per_step": t * 1e3,
                           "parallelism": f"data-parallel x{world} over texel batches of all {M} materials: latents "
                                          "sharded by row bands, batched halo all-to-alls, one stacked all-reduce "
                                          f"of {M} x [dW | loss] ({M * (ntc.ntc_num_params(d) + 1) * 4} B)",
                           "workload": f"per step and rank: 4 x 256^2 crops per material in the rank's band",
                           "gpu_launches_per_step": dp.launches}
    return res


def screen_queries(n_mats, block=64, sw=3840, sh=2160, seed=SEED_BASE + 40):
    """Table 4 analog: a full-screen quad at 3840x2160 sampling mip 0 of a 4096^2
    texture, queries in screen (row-major) order; every 64x64 screen block shows one of
    `n_mats` materials (seeded), so material runs are long but interleaved across the frame."""
    py, px = np.meshgrid(np.arange(sh), np.arange(sw), indexing="ij")
    x = ((px.astype(np.int64) * 2 + 1) * W) // (2 * sw)
    y = ((py.astype(np.int64) * 2 + 1) * W) // (2 * sh)
    xym = np.stack([x.ravel(), y.ravel(), np.zeros(x.size, np.int64)], 1).astype(np.int32)
    tab = np.random.default_rng(seed).integers(0, n_mats, ((sh + block - 1) // block, (sw + block - 1) // block))
    mid = tab[py // block, px // block].ravel().astype(np.int32)
    return xym, mid


def bench_multi(args, ntc, torch, dev, flush, n_mats=8):
    """f3: the Table 4 screen workload (8,294,400 mip-0 queries in screen order) over 8 materials
    (4096^2, 8 channels, NTC 0.2), one ntc_decode_texels_multi call (device bucketing + one
    persistent decode launch); also the worst case (material uniformly random per query) and
    the same screen queries on a single material through ntc_decode_texels."""
    d = Profile.named("ntc0.2", W, 8)
    mats = []
    for k in range(n_mats):
        seed = SEED_BASE + 4 + k  # configs[4]: per-material seed = base + material id
        mats.append(ntc.Material(d, torch.from_numpy(gen_codes(seed, ntc.grid_list(d))).to(dev),
                                 torch.from_numpy(gen_weights_f16(seed + 1, d.input_dim, 8).view(np.int16)).to(dev)))
    xym, mid = screen_queries(n_mats)
    n = xym.shape[0]
    reps = max(3, min(args.steps, 10))
    xym_d = torch.from_numpy(xym).to(dev)
    q = ntc.pack_queries(xym_d, torch.from_numpy(mid).to(dev))
    qr = ntc.pack_queries(xym_d, torch.from_numpy(
        np.random.default_rng(SEED_BASE + 41).integers(0, n_mats, n).astype(np.int32)).to(dev))
    q1 = ntc.pack_queries(xym_d)
    out = torch.empty((n, 8), dtype=torch.float16, device=dev)
    scratch = torch.empty(ntc.ntc_decode_multi_scratch_bytes(n), dtype=torch.uint8, device=dev)
    t = _device_time(torch, lambda: ntc.ntc_decode_texels_multi(mats, q, out, scratch=scratch), flush, reps)
    tr = _device_time(torch, lambda: ntc.ntc_decode_texels_multi(mats, qr, out, scratch=scratch), flush, reps)
    t1 = _device_time(torch, lambda: ntc.ntc_decode_texels(mats[0], q1, out), flush, reps)
    return {"metric": "multi-material decoded Gtexel/s", "value": n / t / 1e9, "unit": UNIT,
            "workload": f"Table 4 analog: 3840x2160 screen-order mip-0 queries ({n}), {n_mats} x 4096^2 x 8ch "
                        "NTC0.2 materials, one material per 64x64 screen block",
            "ms_per_step": t * 1e3, "gpu_launches_per_step": 5,
            "random_material_per_query": {"value": n / tr / 1e9, "ms_per_step": tr * 1e3},
            "single_material_same_queries": {"value": n / t1 / 1e9, "ms_per_step": t1 * 1e3}}


def chain_part_texels(ntc, d, nparts):
    """Texel range [lo, hi) of every ntc_decode_chain_part part in the dense chain layout:
    parts split the chain's 128-texel tiles evenly (tiles never straddle mips)."""
    M = ntc.ntc_num_mips(d)
    starts, t = [], 0
    for m in range(M):
        starts.append(t)
        t += -(-(d.width >> m) ** 2 // 128)
    starts.append(t)

    def texel(tile):
        for m in range(M):
            if tile < starts[m + 1]:
                return ntc.ntc_mip_offset(d, m) + min((tile - starts[m]) * 128, (d.width >> m) ** 2)
        return ntc.ntc_chain_texels(d)

    return [(texel(t * p // nparts), texel(t * (p + 1) // nparts)) for p in range(nparts)]


def e2e(args, ntc, torch, d, codes, wts, dev, world, nparts=8):
    """Same metric through the public API: H2D of the compressed material (codes + fp16
    weights) from pinned memory, material create (pack), full-chain decode, D2H of the
    decoded chain into pinned memory, every step.  The decode runs as `nparts`
    ntc_decode_chain_part launches and each part's D2H copy starts on a copy stream as soon
    as that part is decoded, so the PCIe read-back overlaps the decode."""
    T, c = ntc.ntc_chain_texels(d), d.channels
    h_codes = torch.from_numpy(codes).pin_memory()
    h_w = torch.from_numpy(wts.view(np.int16)).pin_memory()
    h_out = torch.empty((T * c,), dtype=torch.float16).pin_memory()
    d_codes = torch.empty_like(h_codes, device=dev)
    d_w = torch.empty_like(h_w, device=dev)
    d_out = torch.empty((T * c,), dtype=torch.float16, device=dev)
    s = torch.cuda.current_stream()
    cs = torch.cuda.Stream(device=dev)
    ranges = chain_part_texels(ntc, d, nparts)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    evp = [torch.cuda.Event() for _ in range(nparts)]
    steps = max(1, min(args.steps, 10))
    tot = 0.0
    for i in range(steps + 1):
        e0.record(s)
        d_codes.copy_(h_codes, non_blocking=True)
        d_w.copy_(h_w, non_blocking=True)
        m = ntc.Material(d, d_codes, d_w)
        for p, (lo, hi) in enumerate(ranges):
            ntc.ntc_decode_chain_part(m, p, nparts, d_out)
            evp[p].record(s)
            cs.wait_event(evp[p])
            with torch.cuda.stream(cs):
                h_out[lo * c: hi * c].copy_(d_out[lo * c: hi * c], non_blocking=True)
        e1.record(cs)
        e1.synchronize()
        m.close()
        if i > 0:
            tot += e0.elapsed_time(e1) / 1e3
    return {"value": T * world * steps / tot / 1e9, "unit": UNIT,
            "h2d_bytes_per_step": int(h_codes.numel() + 2 * h_w.numel()),
            "d2h_bytes_per_step": int(2 * h_out.numel()),
            "note": f"decode via ntc_material_create + {nparts} ntc_decode_chain_part launches, each part's D2H "
                    "overlapped on a copy stream; host-pinned in/out"}


# ------------------------------------------------------------------------------------ oracle
def _oracle_decode_sample(O, d, codes, wts, n, seed):
    q = gen_queries(seed, W, n, "area")
    t0 = time.perf_counter()
    O.decode_texels(d, codes, wts, q, nthreads=0)
    return time.perf_counter() - t0


def cpu_baseline(d, codes, wts, budget_s=15.0):
    import oracle as O

    O.build()
    n, el = 1 << 14, 0.0
    while True:
        el = _oracle_decode_sample(O, d, codes, wts, n, 77)
        if el >= budget_s / 3 or n >= (1 << 24):
            break
        n *= 2
    cores = os.cpu_count()
    return {"value": n / el / 1e9, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"{n} area-uniform random texels of the 4096^2 9ch chain, oracle decode_texels "
                      f"(C fp64, OpenMP {cores} threads), {el:.2f} s",
            "protocol": oracle_protocol(O)}


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def _oracle_codes(O, d, seed):
    grids = []
    for j in range(O.num_levels(d)):
        r0, r1 = O.grid_res(d, j)
        grids += [(r0 * r0 * d.c0, d.b0), (r1 * r1 * d.c1, d.b1)]
    return gen_codes(seed, grids)


def oracle_protocol(O):
    """SURVEY.md 8(d) oracle timing: the CPU model, C1 (256^2 x 8ch mip 0) on ONE core, the full
    C2 chain (2048^2 x 9ch, 5,592,405 texels) and one C4 training step (4 x 256^2 crops at LOD 0
    of the 4096^2 9ch material: loss + every gradient) on all host cores.  Reported only."""
    out = {"cpu_model": _cpu_model(), "cores": os.cpu_count()}
    d1 = Profile.named("ntc0.2", 256, 8)
    c1, w1 = _oracle_codes(O, d1, SEED_BASE + 0), gen_weights_f16(SEED_BASE + 1, d1.input_dim, 8)
    t0 = time.perf_counter()
    O.decode_mip(d1, c1, w1, 0, nthreads=1)
    out["C1_single_core_s"] = round(time.perf_counter() - t0, 3)
    d2 = Profile.named("ntc0.2", 2048, 9)
    c2, w2 = _oracle_codes(O, d2, SEED_BASE + 1), gen_weights_f16(SEED_BASE + 2, d2.input_dim, 9)
    t0 = time.perf_counter()
    for m in range(O.num_mips(2048)):
        O.decode_mip(d2, c2, w2, m, nthreads=os.cpu_count())
    el = time.perf_counter() - t0
    out["C2_full_chain_s"] = round(el, 3)
    out["C2_Gtexel_s"] = round(5592405 / el / 1e9, 6)
    d4 = Profile.named("ntc0.2", W, C)
    NL = sum(r0 * r0 * d4.c0 + r1 * r1 * d4.c1 for r0, r1 in (O.grid_res(d4, j) for j in range(O.num_levels(d4))))
    lat = gen_latents(SEED_BASE + 6, NL)
    par = gen_weights_f32(SEED_BASE + 7, d4.input_dim, C)
    ref = u8_to_f16_bits(gen_reference_u8(SEED_BASE + 4, W, C))
    crops = gen_crops(SEED_BASE + 3, W, 0, 4, 256)
    t0 = time.perf_counter()
    O.train_grads(d4, lat, par, 0, crops, ref, 7, 1, nthreads=os.cpu_count())
    el = time.perf_counter() - t0
    out["C4_step_s"] = round(el, 3)
    out["C4_texels_s"] = round(4 * 256 * 256 / el, 1)
    return out


def run_reference(args, rank, world):
    """--impl reference: the CPU oracle as it stands, on the host cores, same metric/config."""
    if rank != 0:
        return None
    import oracle as O

    O.build()
    d = Profile.named("ntc0.2", W, C)
    grids = []
    for j in range(O.num_levels(d)):
        r0, r1 = O.grid_res(d, j)
        grids += [(r0 * r0 * d.c0, d.b0), (r1 * r1 * d.c1, d.b1)]
    codes = gen_codes(SEED_BASE + 4, grids)
    wts = gen_weights_f16(SEED_BASE + 5, d.input_dim, C)
    n = 1 << 16
    for i in range(args.warmup):
        _oracle_decode_sample(O, d, codes, wts, n, 1000 + i)
    tot = 0.0
    for i in range(args.steps):
        tot += _oracle_decode_sample(O, d, codes, wts, n, 2000 + i)
    v = n * args.steps / tot / 1e9
    cores = os.cpu_count()
    return {"metric": METRIC, "value": v, "unit": UNIT, "impl": "reference", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot / args.steps * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": WORKLOAD + f" (bounded sample: {n} texels/step)"},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": f"{n} area-uniform random texels per step, C fp64 oracle, OpenMP"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--no-extras", action="store_true", help="skip the random-access and multi-material lines")
    ap.add_argument("--no-c5", action="store_true", help="skip the 64-material configs[4] lines")
    ap.add_argument("--c5-materials", type=int, default=64, help="materials of the configs[4] lines (64)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        res = run_reference(args, rank, world)
        if res is not None:
            print(json.dumps(res), flush=True)
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        dev = torch.device("cuda", local_rank % torch.cuda.device_count())
        torch.cuda.set_device(dev)
        backend = os.environ.get("NTC_BENCH_BACKEND", "nccl")  # gloo: several ranks sharing one GPU (tests)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    res = run_ours(args, rank, world, local_rank)
    if rank == 0:
        print(json.dumps(res), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
