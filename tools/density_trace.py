"""Density trajectory of the MiCRO threshold controller (alpha = 0.01) on
fresh N(0,1) gradients: windowed mean density over many iterations."""
import os
import statistics
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2310_00967_b200 import engine  # noqa: E402

n_g = int(sys.argv[1]) if len(sys.argv) > 1 else 11_700_000
d = float(sys.argv[2]) if len(sys.argv) > 2 else 0.01
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 12000
delta0 = statistics.NormalDist().inv_cdf(1 - d / 2) * 0.01
m = engine.Micro(n_g, 1, density=d, initial_threshold=delta0, dense_output=False)
g = torch.empty(n_g, device="cuda")
Ks = []
for t in range(iters):
    engine.synth_gaussian(g, 1, 0, t)
    m.step([g], 0.01, t)
    if (t + 1) % 4000 == 0:
        h = m.history(4000)
        Ks.append(h["K"])
K = np.concatenate(Ks) / n_g
for a in range(0, len(K), 500):
    w = K[a:a + 500]
    print(f"t={a:6d}..{a + 500:6d}  mean density {w.mean() * 100:.4f} %  rel {w.mean() / d - 1:+.3f}")
