"""One process driving all n ranks (micro_group_*): n rank contexts — here
all on cuda:0, each with its own stream — exchange over direct peer pointers
with event barriers.  Bit-exact against the oracle cluster.  GPU only."""
import numpy as np
import pytest
import torch

from oracle import Oracle, OracleCluster

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2310_00967_b200.dist import GroupMicro


@pytest.mark.parametrize("n,n_g,ef", [(2, 100_003, True), (4, 65_536, True), (3, 20_000, False)])
def test_group_step_matches_oracle(n, n_g, ef):
    o = Oracle()
    d, delta0, eta = 0.02, 0.015, 0.01
    g = GroupMicro(n_g, n, devices=[0] * n, density=d, initial_threshold=delta0, error_feedback=ef)
    xs = [torch.zeros(n_g, device="cuda") for _ in range(n)]
    for m, x in zip(g.ranks, xs):
        m.set_model(x)
    ref = OracleCluster(n_g, n, density=d, delta0=delta0, error_feedback=ef, model=True)
    for t in range(10):
        G = np.stack([o.gaussian(5, i, t, n_g) for i in range(n)])
        Gd = [torch.from_numpy(G[i]).cuda() for i in range(n)]
        torch.cuda.synchronize()
        g.step(Gd, eta, t)
        r = ref.step(G, eta, t)
        g.synchronize()
        for rank, m in enumerate(g.ranks):
            idx, sums = m.union()
            assert np.array_equal(idx, r["union_idx"]), (t, rank)
            assert np.array_equal(sums, r["union_sum"]), (t, rank)
            assert np.array_equal(m.residual(0), ref.e[rank]), (t, rank)
            assert m.query().deltas[0] == r["delta_next"][rank]
            assert np.array_equal(xs[rank].cpu().numpy(), ref.x), (t, rank)
    g.close()


def _group_cases(count=24, seed=77):
    rng = np.random.default_rng(seed)
    return [(int(rng.integers(2, 9)), int(rng.choice([17, 4099, 70_001, 300_007])) + int(rng.integers(0, 50)),
             float(rng.choice([0.001, 0.02, 0.2])), bool(rng.integers(0, 4)), bool(rng.integers(0, 2)))
            for _ in range(count)]


@pytest.mark.parametrize("n,n_g,d,ef,norm", _group_cases())
def test_group_sweep(n, n_g, d, ef, norm):
    """Ragged sizes, 2-8 ranks, error norm on/off: the peer exchange (bulk)
    through the group mode, bit-exact against the oracle cluster."""
    n_g = max(n_g, n)
    o = Oracle()
    g = GroupMicro(n_g, n, devices=[0] * n, density=d, initial_threshold=0.01, error_feedback=ef,
                   record_error_norm=norm)
    ref = OracleCluster(n_g, n, density=d, delta0=0.01, error_feedback=ef)
    for t in range(4):
        G = np.stack([o.gaussian(9, i, t, n_g) for i in range(n)])
        Gd = [torch.from_numpy(G[i]).cuda() for i in range(n)]
        torch.cuda.synchronize()
        g.step(Gd, 0.01, t)
        r = ref.step(G, 0.01, t)
        g.synchronize()
        for rank, m in enumerate(g.ranks):
            idx, sums = m.union()
            assert np.array_equal(idx, r["union_idx"]) and np.array_equal(sums, r["union_sum"]), (t, rank)
            assert np.array_equal(m.residual(0), ref.e[rank]), (t, rank)
    g.close()
