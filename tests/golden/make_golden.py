"""Regenerate tests/golden/*.npz from the reference's own compiled code
(oracle/_ref/libsparsim_ref.so, built from /root/reference by oracle/Makefile).

Each fixture is a whole MiCRO run (harness.cpp:121-224 order, fp64) on the
synthetic gradients of include/micro_synth.h (seed 7, upcast to fp64):
per-iteration counts, union indices, reduced sums, thresholds used / next,
and the final residuals and model.  Run:  python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
from oracle import Oracle, RefCluster  # noqa: E402

CASES = {
    # name: (n_g, n, d, delta0, full, ef, iters)
    "n1_d01": (10_000, 1, 0.01, 0.01, False, True, 30),
    "n2_rem": (10_007, 2, 0.01, 0.02, False, True, 30),
    "n3_d05": (9_999, 3, 0.05, 0.01, False, True, 20),
    "n8_d02": (12_345, 8, 0.02, 0.01, False, True, 20),
    "n4_noef": (8_000, 4, 0.01, 0.01, False, False, 12),
    "n4_full": (8_000, 4, 0.01, 0.01, True, True, 12),
}
SEED, ETA = 7, 0.01


def make(name, n_g, n, d, delta0, full, ef, iters):
    o = Oracle()
    ref = RefCluster(n_g, n, d, delta0, 0.01, 1e-12, full, ef, model=True)
    rec = dict(counts=[], union_idx=[], union_sum=[], delta_used=[], delta_next=[])
    for t in range(iters):
        G = np.stack([o.gaussian(SEED, i, t, n_g) for i in range(n)]).astype(np.float64)
        r = ref.step(G, ETA, t)
        for k in rec:
            rec[k].append(r[k])
    K = np.array([u.size for u in rec["union_idx"]], np.int64)
    np.savez_compressed(
        os.path.join(HERE, f"micro_ref64_{name}.npz"),
        config=np.array([n_g, n, d, delta0, int(full), int(ef), iters, SEED, ETA], np.float64),
        counts=np.stack(rec["counts"]), K=K,
        union_idx=np.concatenate(rec["union_idx"]).astype(np.int64),
        union_sum=np.concatenate(rec["union_sum"]),
        delta_used=np.stack(rec["delta_used"]), delta_next=np.stack(rec["delta_next"]),
        residuals=ref.residuals(), model=ref.x)


if __name__ == "__main__":
    for name, cfg in CASES.items():
        make(name, *cfg)
        print("wrote", name)
