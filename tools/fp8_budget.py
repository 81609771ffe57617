"""f4 FP8 check (profiling helper, not product code): decode error of lower-precision hidden
activations against the exact fp64 MLP, on 200,000 random fp16 inputs of an
NTC 0.2, 9-channel material with the bench's weight recipe.  The decode bar is max |err| <=
2e-3 (BASELINE.json north_star).  usage: python tools/fp8_budget.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2305_17105_b200.synth import Profile, gen_weights_f16  # noqa: E402


def main():
    d = Profile.named("ntc0.2", 256, 9)
    D = d.input_dim
    w = gen_weights_f16(5, D, 9).view(np.float16).astype(np.float64)
    o = 0
    W1 = w[o:o + 64 * D].reshape(64, D); o += 64 * D
    b1 = w[o:o + 64]; o += 64
    W2 = w[o:o + 4096].reshape(64, 64); o += 4096
    b2 = w[o:o + 64]; o += 64
    W3 = w[o:o + 64 * 9].reshape(9, 64); o += 64 * 9
    b3 = w[o:o + 9]
    X = np.random.default_rng(0).uniform(-0.5, 0.5, (200000, D))
    X = torch.tensor(X).to(torch.float16).double().numpy()

    def hg(z):
        return np.where(z < -1.5, 0, np.where(z > 1.5, z, z / 3 * (z + 1.5)))

    def q(a, dt):
        return a if dt is None else torch.tensor(a).to(dt).double().numpy()

    def run(dt):
        h1 = q(hg(q(X, dt) @ W1.T + b1), dt)
        h2 = q(hg(h1 @ W2.T + b2), dt)
        return np.clip(h2 @ W3.T + b3, 0, 1)

    ref = run(None)
    for name, dt in [("fp16 activations (the shipped path)", torch.float16),
                     ("e4m3 activations (kind::f8f6f4)", torch.float8_e4m3fn),
                     ("e5m2 activations", torch.float8_e5m2)]:
        err = np.abs(run(dt) - ref)
        print(f"{name:38s} max {err.max():.2e}  p99.9 {np.quantile(err, 0.999):.2e}  "
              f"{'within' if err.max() <= 2e-3 else 'OUTSIDE'} the 2e-3 bar")


if __name__ == "__main__":
    main()
