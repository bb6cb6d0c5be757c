"""The comparison sparsifiers on the GPU (csrc/baselines.cuh; run_iteration's
top-k / CLT-k / hard-threshold / dense branches, harness.cpp:152-224,
SURVEY.md §8f-3) against the oracle: fp32 vs the numpy restatement
(BaselineCluster, itself pinned to the reference's code) and fp64 vs the
reference's own code, bit for bit — counts, union, sums, residuals, model,
dense g/n and records, with and without magnitude ties.  GPU only."""
import numpy as np
import pytest
import torch

from oracle import BaselineCluster, Oracle, RefCluster

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2310_00967_b200 import engine


def grads(rng, n, n_g, t, ties, dtype):
    if ties:  # few distinct magnitudes: the tie rule (lower index) decides top-k
        return (rng.integers(-4, 5, size=(n, n_g)).astype(np.float64) / 4.0).astype(dtype)
    return rng.standard_normal((n, n_g)).astype(dtype)


def run(kind, n_g, n, d, ties, dtype=np.float32, ef=True, iters=6, delta0=0.02, split=False):
    rng = np.random.default_rng(n_g * 7 + n)
    tdt = torch.float32 if dtype == np.float32 else torch.float64
    m = engine.Micro(n_g, n, dtype=tdt, density=d, initial_threshold=delta0, error_feedback=ef, sparsifier=kind)
    x = torch.zeros(n_g, dtype=tdt, device="cuda")
    m.set_model(x)
    if dtype == np.float64:
        ref = RefCluster(n_g, n, d, delta0, 0.01, 1e-12, False, ef, model=True)
        step = lambda G, t: ref.step(G, 0.01, t, kind=kind)  # noqa: E731
        resid = ref.residuals
    else:
        ref = BaselineCluster(n_g, n, kind, density=d, delta0=delta0, error_feedback=ef, dtype=np.float32,
                              model=True)
        step = lambda G, t: ref.step(G, 0.01, t)  # noqa: E731
        resid = lambda: ref.e  # noqa: E731
    k_glob = Oracle().global_target_count(d, n_g)
    for t in range(iters):
        G = grads(rng, n, n_g, t, ties, dtype)
        if split:  # micro_compress + micro_aggregate
            m.compress(list(torch.from_numpy(G).cuda()), 0.01, t)
            m.aggregate()
        else:
            m.step(list(torch.from_numpy(G).cuda()), 0.01, t)
        r = step(G, t)
        st = m.query()
        idx, sums = m.union()
        assert np.array_equal(st.counts, r["counts"]), (t, st.counts, r["counts"])
        assert np.array_equal(idx.astype(np.int64), r["union_idx"]), t
        assert np.array_equal(sums, r["union_sum"].astype(sums.dtype)), t
        res = np.stack([m.residual(i) for i in range(n)])
        assert np.array_equal(res, resid().astype(res.dtype)), t
        assert np.array_equal(x.cpu().numpy(), ref.x.astype(res.dtype)), t
        dw = np.zeros(n_g, res.dtype)
        dw[r["union_idx"]] = (r["union_sum"] / n).astype(res.dtype) if dtype == np.float64 else \
            (r["union_sum"].astype(np.float32) / np.float32(n))
        assert np.array_equal(m.dense(), dw), t
    recs = m.records(iters)
    for rec in recs:  # harness.cpp:135, :170, :226-236
        assert rec["threshold"] == (delta0 if kind == "hard" else 0.0)
        assert rec["buildup_factor"] == (rec["K"] / k_glob if rec["total_selected"] else 0.0)
    m.close()
    return [rec["K"] for rec in recs]


@pytest.mark.parametrize("kind", ["topk", "cltk", "hard", "dense"])
@pytest.mark.parametrize("n_g,n,d,ties", [(10_000, 1, 0.01, False), (20_011, 3, 0.02, False),
                                          (8_192, 4, 0.05, True), (300_007, 2, 0.003, True), (1_000, 2, 1.0, False)])
def test_gpu_baselines_f32(kind, n_g, n, d, ties):
    run(kind, n_g, n, d, ties)


@pytest.mark.ref
@pytest.mark.parametrize("kind", ["topk", "cltk", "hard", "dense"])
@pytest.mark.parametrize("n_g,n,d,ties", [(5_003, 2, 0.02, False), (4_096, 3, 0.05, True)])
def test_gpu_baselines_f64_reference_code(kind, n_g, n, d, ties):
    run(kind, n_g, n, d, ties, dtype=np.float64)


@pytest.mark.parametrize("kind", ["topk", "hard"])
def test_gpu_baselines_ef_off(kind):
    run(kind, 12_345, 2, 0.01, False, ef=False)


def test_gpu_topk_large_ties():
    """Ties spread over many 65536-way chunks: the tie index search."""
    run("topk", 2_000_003, 1, 0.0007, True, iters=3)


@pytest.mark.parametrize("kind", ["topk", "cltk", "hard"])
@pytest.mark.parametrize("n_g,d,ties,dtype,ef,split", [
    (8_192, 0.05, True, np.float32, True, False),     # the tie rule on the one-worker path
    (10_007, 1.0, False, np.float32, True, False),    # everything selected (top-k's k >= n_g path)
    (4_096, 0.05, True, np.float64, True, False),     # the reference's own code
    (9_999, 0.02, False, np.float32, False, False),   # EF off (top-k / CLT-k: the general path)
    (9_999, 0.02, True, np.float32, True, True),      # micro_compress + micro_aggregate
])
def test_gpu_baselines_one_worker(kind, n_g, d, ties, dtype, ef, split):
    """n = 1: the selection is the union and the single-worker step finishes
    it (k1_stream + k1_gather, as for MiCRO): bit-exact like the general path."""
    run(kind, n_g, 1, d, ties, dtype=dtype, ef=ef, split=split)


# The union of overlapping selections takes one of two device paths, chosen
# on the device from the scan's total K: above 15 % of n_g one pass over the
# bitmap's words (k_union_words), else the ordered emission and a gather per
# entry (k_bitmap_emit + k_union_reduce).  Both against the oracle, with the
# density checked to sit on the intended side (or to cross it mid-run).
@pytest.mark.parametrize("delta0,dense", [(0.0005, True), (0.03, False), (0.0258, False)])
@pytest.mark.parametrize("ef", [True, False])
def test_gpu_union_paths_hard_n8(delta0, dense, ef):
    n_g = 50_021
    Ks = run("hard", n_g, 8, 0.01, False, ef=ef, delta0=delta0)
    if dense:
        assert all(K > 0.15 * n_g for K in Ks), Ks
    else:  # sparse steps first; with EF the union densifies, so both paths run in one context
        assert any(K <= 0.15 * n_g for K in Ks), Ks


@pytest.mark.ref
@pytest.mark.parametrize("delta0", [0.0005, 0.03])
def test_gpu_union_paths_hard_f64_reference_code(delta0):
    run("hard", 20_011, 5, 0.01, False, dtype=np.float64, delta0=delta0)


# Top-k on several workers runs every worker's radix select in shared
# launches (blockIdx.y = worker): ties across many tie-count chunks, up to 8
# workers, fp32 and fp64 (the reference's code).
@pytest.mark.parametrize("n_g,n,d,ties", [(65_537, 8, 0.02, True), (300_007, 5, 0.01, True),
                                          (40_000, 8, 0.3, False)])
def test_gpu_topk_batched_workers(n_g, n, d, ties):
    run("topk", n_g, n, d, ties)


@pytest.mark.ref
def test_gpu_topk_batched_workers_f64_reference_code():
    run("topk", 9_001, 6, 0.03, True, dtype=np.float64)
