"""Per-phase cycle timeline of the training kernel (profiling helper, not product code).

Builds a separate library with -DNTC_TRAIN_TRACE (the MMA-issuing thread of every slot stamps
clock64() at each phase boundary of every tile), runs the bench's C4 step, and prints the mean
cycles of each phase plus the spread over CTAs.  usage: python tools/trace_train.py [--build-only]"""
from __future__ import annotations

import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
PKG = os.path.join(ROOT, "paper_2305_17105_b200")
TDIR = os.path.join(PKG, "build_trace")
TLIB = os.path.join(TDIR, "libntc_trace.so")

PHASES = ["assemble X", "Z1 MMA", "H1 epilogue", "Z2 MMA", "H2 epilogue", "Y MMA", "loss", "dH2 MMA",
          "delta2", "dH1 MMA", "delta1", "dX+dW MMA", "scatter"]


def build():
    from paper_2305_17105_b200 import build as B

    B.build()
    os.makedirs(TDIR, exist_ok=True)
    obj = os.path.join(TDIR, "train.o")
    extra = [a for a in sys.argv[1:] if a.startswith("-D")]
    subprocess.check_call([B.NVCC, *B.FLAGS, "-DNTC_TRAIN_TRACE", *extra, "-c", "-o", obj,
                           os.path.join(PKG, "csrc", "train.cu")])
    objs = [os.path.join(B.OBJDIR, f) for f in os.listdir(B.OBJDIR) if f.endswith(".o") and f != "train.o"]
    subprocess.check_call([B.NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", TLIB, obj, *objs])


def run():
    import ctypes

    import numpy as np
    import torch

    import paper_2305_17105_b200 as ntc

    ntc.LIB_PATH = sys.argv[sys.argv.index("--lib") + 1] if "--lib" in sys.argv else TLIB
    L = ntc.lib()
    from paper_2305_17105_b200.synth import (SEED_BASE, Profile, gen_crops, gen_latents, gen_reference_u8,
                                             gen_weights_f32, u8_to_f16_bits)

    dev = "cuda:0"
    W, C = 4096, 9
    d = Profile.named("ntc0.2", W, C)
    NL, P = ntc.ntc_num_latents(d), ntc.ntc_num_params(d)
    t = {k: torch.zeros(NL, device=dev) for k in ("m_lat", "v_lat", "grad_lat", "noisy")}
    t.update({k: torch.zeros(P, device=dev) for k in ("m_par", "v_par", "grad_par")})
    t["latents"] = torch.from_numpy(gen_latents(SEED_BASE + 6, NL)).to(dev)
    t["params"] = torch.from_numpy(gen_weights_f32(SEED_BASE + 7, d.input_dim, C)).to(dev)
    ref = torch.from_numpy(u8_to_f16_bits(gen_reference_u8(SEED_BASE + 4, W, C)).view(np.int16)).to(dev)
    tr, bufs, loss = ntc.Trainer(d), ntc.make_buffers(t), torch.zeros(1, device=dev)
    crops = gen_crops(SEED_BASE + 3, W, 0, 4, 256)
    nsm = torch.cuda.get_device_properties(0).multi_processor_count
    slots = int(sys.argv[sys.argv.index("--slots") + 1]) if "--slots" in sys.argv else 2
    wps = 8
    buf = torch.zeros(nsm * slots * 16 * wps * 32, dtype=torch.int32, device=dev)
    L.ntc_trace_set.argtypes = [ctypes.c_void_p]
    for i in range(4):
        if i == 3:
            L.ntc_trace_set(buf.data_ptr())
        ntc.ntc_train_step(tr, bufs, ntc.make_batch(0, crops, ref, W * C),
                           ntc.Hparams(0.01, 0.005, 0.9, 0.999, 1e-8, i + 1, 7, 1, 0), loss)
    torch.cuda.synchronize()
    arr = buf.cpu().numpy().astype(np.int64).reshape(nsm, slots, 16, wps, 32) & 0xFFFFFFFF
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    np.save(os.path.join(ROOT, "gpurun_out", "train_trace.npy"), arr)
    report(arr)


# stamp sequence of one tile: k = after phase boundary k, 16 + k = arrival at the barrier ending phase k
SEQ = [(0, "top"), (17, "assemble"), (1, "bar"), (2, "Z1 wait (+fetch)"), (19, "H1 epi"), (3, "bar"),
       (4, "Z2 wait"), (21, "H2 epi"), (5, "bar"), (6, "Y wait"), (23, "loss"), (7, "bar"), (8, "dH2 wait"),
       (25, "delta2"), (9, "bar"), (10, "dH1 wait"), (27, "delta1"), (11, "bar"), (12, "dX wait (+dW issue)"),
       (15, "scatter")]


def report(a):
    import numpy as np

    nsm, slots, iters, wps, _ = a.shape
    segs = np.zeros((len(SEQ) - 1, wps))
    n = 0
    spans = []
    for b in range(nsm):
        for s in range(slots):
            for it in range(iters - 2):
                row = a[b, s, it]
                if row[0, 0] == 0:
                    continue
                v = row[:, [k for k, _ in SEQ]]  # [warp][seq]
                segs += (np.diff(v, axis=1) % (1 << 32)).T
                n += 1
                spans.append(((v[:, -1] - v[:, 0]) % (1 << 32)).max())
    segs /= max(n, 1)
    print(f"tiles traced: {n}; mean tile span {np.mean(spans):.0f} cycles")
    print("segment (ends at)        " + " ".join(f"  w{w}" for w in range(wps)) + "   max")
    for i in range(len(SEQ) - 1):
        print(f"  {SEQ[i + 1][1]:22s}" + " ".join(f"{x:5.0f}" for x in segs[i]) + f" {segs[i].max():5.0f}")
    k = a[:, :, 15]  # [cta][slot][warp][32]
    pro = ((k[..., 1] - k[..., 0]) % (1 << 32)).max(axis=(1, 2))
    loop = ((k[..., 2] - k[..., 1]) % (1 << 32)).max(axis=(1, 2))
    fin = ((k[..., 3] - k[..., 2]) % (1 << 32)).max(axis=(1, 2))
    print(f"per CTA cycles: prologue {pro.mean():.0f} (max {pro.max():.0f}), loop {loop.mean():.0f} "
          f"(min {loop.min():.0f} max {loop.max():.0f}), final {fin.mean():.0f} (max {fin.max():.0f})")
    f = a[:, 0, 14, 0, :8]  # fused-step stamps (thread 0 per CTA), if any
    if f[:, 0].any():
        t0 = f[:, 0].min()
        rel = (f - t0) % (1 << 32)
        names = ["entry", "prep done", "grid sync 1", "train_body done", "grid sync 2", "weights reduce+Adam",
                 "latent Adam"]
        print("fused step, ns from the first CTA entry (mean / max over CTAs):")
        for i, nm in enumerate(names):
            print(f"  {nm:20s} {rel[:, i].mean():9.0f} {rel[:, i].max():9.0f}")
    g0 = k[..., 4].reshape(nsm, -1)
    g1 = k[..., 5].reshape(nsm, -1)
    t0 = g0.min()
    ent = (g0.min(axis=1) - t0) % (1 << 32)
    ex = (g1.max(axis=1) - t0) % (1 << 32)
    print(f"globaltimer ns from first CTA entry: entry spread max {ent.max():.0f}, exit mean {ex.mean():.0f} "
          f"min {ex.min():.0f} max {ex.max():.0f}")
    cta = []
    for b in range(nsm):
        v = a[b, :, :-1][..., [0, 15]].reshape(-1)
        v = v[v > 0]
        if v.size:
            cta.append((v.max() - v.min()) % (1 << 32))
    print(f"CTA loop span cycles: mean {np.mean(cta):.0f} min {np.min(cta):.0f} max {np.max(cta):.0f}")


if __name__ == "__main__":
    if "--report" in sys.argv:  # re-analyse a saved trace here
        import numpy as np

        report(np.load(sys.argv[sys.argv.index("--report") + 1]))
    elif "--build-only" in sys.argv:
        build()
    else:
        if not os.path.exists(TLIB):
            build()
        run()
