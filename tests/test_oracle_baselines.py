"""Pins the numpy restatement of the comparison sparsifiers (oracle
BaselineCluster, fp64) to the reference's own code (harness.cpp:152-224 over
select_topk / cltk_select / hard_threshold_select / select_all, compiled
verbatim) bit for bit, including ties.  CPU only."""
import numpy as np
import pytest

from oracle import BaselineCluster, RefCluster

pytestmark = pytest.mark.ref


@pytest.mark.parametrize("kind", ["topk", "cltk", "hard", "dense"])
@pytest.mark.parametrize("n_g,n,d,ties", [(1000, 1, 0.05, False), (3001, 3, 0.01, False), (512, 4, 0.1, True),
                                          (97, 2, 0.5, True), (64, 8, 1.0, True)])
@pytest.mark.parametrize("ef", [True, False])
def test_baselines_match_reference(kind, n_g, n, d, ties, ef):
    rng = np.random.default_rng(n_g + n)
    ref = RefCluster(n_g, n, d, 0.02, 0.01, 1e-12, False, ef, model=True)
    orc = BaselineCluster(n_g, n, kind, density=d, delta0=0.02, error_feedback=ef, dtype=np.float64, model=True)
    for t in range(8):
        if ties:  # few distinct magnitudes: top-k's tie rule (lower index) decides
            G = rng.integers(-3, 4, size=(n, n_g)).astype(np.float64) / 2.0
        else:
            G = rng.standard_normal((n, n_g))
        a = ref.step(G, 0.01, t, kind=kind)
        b = orc.step(G, 0.01, t)
        assert np.array_equal(a["counts"], b["counts"]), t
        assert np.array_equal(a["union_idx"], b["union_idx"]), t
        assert np.array_equal(a["union_sum"], b["union_sum"]), t
        assert np.array_equal(ref.residuals(), orc.e), t
        assert np.array_equal(ref.x, orc.x), t
