"""The same density trajectory as tools/density_trace.py, run through the
reference's own code (oracle/_ref, fp64) on the CPU: shows the controller's
stationary density is the reference's behaviour."""
import os
import statistics
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle.oracle import RefCluster  # noqa: E402

n_g = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
d = float(sys.argv[2]) if len(sys.argv) > 2 else 0.01
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 3000
delta0 = statistics.NormalDist().inv_cdf(1 - d / 2) * 0.01
ref = RefCluster(n_g, 1, density=d, delta0=delta0)
rng = np.random.default_rng(1)
K = np.empty(iters)
for t in range(iters):
    K[t] = ref.step(rng.standard_normal(n_g), 0.01, t)["counts"][0]
K /= n_g
for a in range(0, iters, 500):
    w = K[a:a + 500]
    print(f"t={a:6d}..{a + 500:6d}  mean density {w.mean() * 100:.4f} %  rel {w.mean() / d - 1:+.3f}")
