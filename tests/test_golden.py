"""The oracle against the committed golden runs of the reference
(tests/golden/*.npz, made by tests/golden/make_golden.py from oracle/_ref).
Runs without /root/reference.  CPU only."""
import glob
import os

import numpy as np
import pytest

from oracle import Oracle, OracleCluster

GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "micro_ref64_*.npz")))


def load(path):
    z = np.load(path)
    n_g, n, d, delta0, full, ef, iters, seed, eta = z["config"].tolist()
    return z, dict(n_g=int(n_g), n=int(n), d=d, delta0=delta0, full=bool(full), ef=bool(ef),
                   iters=int(iters), seed=int(seed), eta=eta)


def replay(cluster, z, c, o, dtype):
    off = 0
    for t in range(c["iters"]):
        G = np.stack([o.gaussian(c["seed"], i, t, c["n_g"]) for i in range(c["n"])]).astype(dtype)
        r = cluster.step(G, c["eta"], t)
        K = int(z["K"][t])
        yield t, r, z["counts"][t], z["union_idx"][off:off + K], z["union_sum"][off:off + K], \
            z["delta_used"][t], z["delta_next"][t]
        off += K


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p)[12:-4] for p in GOLDEN])
def test_oracle_f64_reproduces_golden(path):
    z, c = load(path)
    o = Oracle()
    cl = OracleCluster(c["n_g"], c["n"], c["d"], c["delta0"], 0.01, 1e-12, c["full"], c["ef"],
                       dtype=np.float64, model=True)
    for t, r, cnt, u, s, du, dn in replay(cl, z, c, o, np.float64):
        assert np.array_equal(r["counts"], cnt), t
        assert np.array_equal(r["union_idx"], u), t
        assert np.array_equal(r["union_sum"], s), t
        assert np.array_equal(r["delta_used"], du) and np.array_equal(r["delta_next"], dn), t
    assert np.array_equal(cl.e, z["residuals"])
    assert np.array_equal(cl.x, z["model"])
