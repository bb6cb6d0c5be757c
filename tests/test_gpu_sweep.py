"""Seeded random sweep over shapes the fixed cases miss (partition edges that
cut units and CTA runs, tiny and ragged vectors, many workers, every
sparsifier and mode), each bit-exact against the oracle for a few
iterations.  GPU only."""
import numpy as np
import pytest
import torch

from oracle import BaselineCluster, Oracle, OracleCluster

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2310_00967_b200 import engine


def _cases(count=150, seed=2024):
    rng = np.random.default_rng(seed)
    out = []
    for c in range(count):
        n = int(rng.choice([1, 1, 2, 3, 4, 5, 7, 8, 13]))
        n_g = int(max(n, rng.choice([n, 31, 513, 4097, 8191, 40_961, 200_003]) + int(rng.integers(0, 97))))
        d = float(rng.choice([0.001, 0.01, 0.05, 0.3, 1.0]))
        kind = "micro" if c % 3 else str(rng.choice(["micro", "topk", "cltk", "hard", "dense"]))
        out.append((c, n_g, n, d, bool(rng.integers(0, 4)), kind, bool(rng.integers(0, 2)), float(rng.choice([0.0, 0.01, 0.05]))))
    return out


@pytest.mark.parametrize("case,n_g,n,d,ef,kind,dense,delta0", _cases())
def test_sweep(case, n_g, n, d, ef, kind, dense, delta0):
    o = Oracle()
    m = engine.Micro(n_g, n, density=d, initial_threshold=delta0, error_feedback=ef, sparsifier=kind,
                     dense_output=dense)
    x = torch.zeros(n_g, device="cuda")
    m.set_model(x)
    if kind == "micro":
        ref = OracleCluster(n_g, n, density=d, delta0=delta0, error_feedback=ef, model=True)
    else:
        ref = BaselineCluster(n_g, n, kind, density=d, delta0=delta0, error_feedback=ef, model=True)
    for t in range(4):
        G = np.stack([o.gaussian(case, i, t, n_g) for i in range(n)])
        m.step(list(torch.from_numpy(G).cuda()), 0.01, t)
        r = ref.step(G, 0.01, t)
        idx, sums = m.union()
        assert np.array_equal(m.query().counts, r["counts"]), t
        assert np.array_equal(idx.astype(np.int64), r["union_idx"]), t
        assert np.array_equal(sums, r["union_sum"].astype(np.float32)), t
        assert np.array_equal(np.stack([m.residual(i) for i in range(n)]), ref.e), t
        assert np.array_equal(x.cpu().numpy(), ref.x), t
        if dense:
            dw = np.zeros(n_g, np.float32)
            dw[r["union_idx"]] = r["union_sum"].astype(np.float32) / np.float32(n)
            assert np.array_equal(m.dense(), dw), t
    m.close()


@pytest.mark.ref
@pytest.mark.parametrize("case,n_g,n,d,ef,kind,dense,delta0", _cases(count=40, seed=99))
def test_sweep_f64_reference_code(case, n_g, n, d, ef, kind, dense, delta0):
    """The same sweep in fp64 against the reference's own compiled code."""
    from oracle import RefCluster
    o = Oracle()
    m = engine.Micro(n_g, n, dtype=torch.float64, density=d, initial_threshold=delta0, error_feedback=ef,
                     sparsifier=kind, dense_output=dense)
    x = torch.zeros(n_g, device="cuda", dtype=torch.float64)
    m.set_model(x)
    ref = RefCluster(n_g, n, d, delta0, 0.01, 1e-12, False, ef, model=True)
    for t in range(3):
        G = np.stack([o.gaussian(case, i, t, n_g) for i in range(n)]).astype(np.float64)
        m.step(list(torch.from_numpy(G).cuda()), 0.01, t)
        r = ref.step(G, 0.01, t, kind=kind)
        idx, sums = m.union()
        assert np.array_equal(m.query().counts, r["counts"]), t
        assert np.array_equal(idx.astype(np.int64), r["union_idx"]), t
        assert np.array_equal(sums, r["union_sum"]), t
        assert np.array_equal(np.stack([m.residual(i) for i in range(n)]), ref.residuals()), t
        assert np.array_equal(x.cpu().numpy(), ref.x), t
    m.close()
