"""Chain of trust, link 1: the C restatement in float64 equals the reference's
own compiled code (oracle/_ref) BIT FOR BIT over whole multi-iteration MiCRO
runs.  Link 2 (GPU float32 == restatement float32)
lives in tests/test_gpu_parity.py.  CPU only."""
import numpy as np
import pytest

from oracle import Oracle, OracleCluster, RefCluster

pytestmark = pytest.mark.ref

CASES = [
    # n_g, n, d, delta0, full, ef, iters
    (10_000, 1, 0.01, 0.01, False, True, 40),
    (10_007, 2, 0.01, 0.02, False, True, 40),
    (9_999, 3, 0.05, 0.01, False, True, 30),
    (20_000, 4, 0.01, 0.025, False, True, 30),
    (12_345, 8, 0.02, 0.01, False, True, 30),
    (4_096, 16, 0.01, 0.01, False, True, 20),
    (8_000, 4, 0.01, 0.01, True, True, 20),
    (8_000, 4, 0.01, 0.01, False, False, 20),
    (2_048, 4, 1.0, 0.0, False, True, 10),  # d = 1, delta0 = 0 (test_harness.cpp:60-76)
]


@pytest.mark.parametrize("n_g,n,d,delta0,full,ef,iters", CASES)
def test_restatement_f64_equals_reference(n_g, n, d, delta0, full, ef, iters):
    o = Oracle()
    ref = RefCluster(n_g, n, d, delta0, 0.01, 1e-12, full, ef, model=True)
    orc = OracleCluster(n_g, n, d, delta0, 0.01, 1e-12, full, ef, dtype=np.float64, model=True)
    eta = 0.01
    for t in range(iters):
        G = np.stack([o.gaussian(7, i, t, n_g) for i in range(n)]).astype(np.float64)
        a = ref.step(G, eta, t)
        b = orc.step(G, eta, t)
        for key in ("counts", "union_idx", "union_sum", "delta_used", "delta_next"):
            assert np.array_equal(a[key], b[key]), (t, key)
        # MiCRO never builds up: |union| == sum k_i (acceptance.cpp:93-118)
        assert a["union_idx"].size == a["counts"].sum()
        assert np.array_equal(ref.residuals(), orc.e), t
        assert np.array_equal(ref.x, orc.x), t
        if d == 1.0 and delta0 == 0.0 and t > 0:
            pass
    if d == 1.0 and delta0 == 0.0:
        # density 1, threshold 0: everything nonzero is sent, residual stays 0
        assert np.all(orc.e == 0)


def test_synthetic_gradients_are_gaussian():
    o = Oracle()
    g = o.gaussian(1, 0, 0, 1_000_003)
    assert np.isfinite(g).all()
    assert abs(g.mean()) < 5e-3 and abs(g.std() - 1) < 5e-3
    # 99th percentile of |N(0,1)| is 2.5758
    assert abs(np.quantile(np.abs(g), 0.99) - 2.5758) < 0.02
    # deterministic, keyed by (seed, worker, t)
    assert np.array_equal(g[:1000], o.gaussian(1, 0, 0, 1000))
    assert not np.array_equal(g[:1000], o.gaussian(1, 1, 0, 1000))
    assert not np.array_equal(g[:1000], o.gaussian(1, 0, 1, 1000))
    assert not np.array_equal(g[:1000], o.gaussian(2, 0, 0, 1000))
