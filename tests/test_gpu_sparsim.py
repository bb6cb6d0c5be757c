"""The reference's own unit tests, restated against the value-level CUDA API
(paper_2310_00967_b200.sparsim), plus randomized comparisons with the
reference's compiled code.  GPU only."""
import numpy as np
import pytest
import torch

from oracle import Oracle, Reference

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2310_00967_b200 import sparsim as S
    from paper_2310_00967_b200._lib import InvalidArgument, LogicError


def vec(xs, dtype=torch.float64):
    return torch.tensor(xs, dtype=dtype, device="cuda")


def full(v):
    return S.PartitionRange(0, v.numel(), 0)


# test_sparsifier.cpp:47-69
@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_select_examples(dtype):
    acc = vec([1, -3, 0.5, 2], dtype)
    sel = S.select_by_threshold(acc, full(acc), 1.5)
    assert sel.indices.tolist() == [1, 3] and sel.values.tolist() == [-3, 2]
    assert S.select_by_threshold(acc, full(acc), 100.0).count() == 0
    z = vec([0, -0.25, 0, 7], dtype)
    assert S.select_by_threshold(z, full(z), 0.0).indices.tolist() == [1, 3]
    five = vec([5, 5, 5, 5], dtype)
    assert S.select_by_threshold(five, S.PartitionRange(1, 3, 0), 0.0).indices.tolist() == [1, 2]
    with pytest.raises(InvalidArgument):
        S.select_by_threshold(five, S.PartitionRange(0, 9, 0), 0.0)
    with pytest.raises(ValueError):
        S.select_by_threshold(five, full(five), -1.0)
    assert S.hard_threshold_select(vec([0.1, 0.9, 0.5], dtype), 0.4).indices.tolist() == [1, 2]


@pytest.mark.ref
def test_select_randomized_vs_reference():
    ref = Reference()
    o = Oracle()
    rng = np.random.default_rng(13)
    for rep in range(200):
        n_g = int(rng.integers(1, 300_000)) if rep % 10 == 0 else int(rng.integers(1, 20_000))
        acc = rng.standard_normal(n_g)
        s = int(rng.integers(0, n_g))
        e = int(rng.integers(s, n_g + 1))
        d = float(rng.uniform(0, 2.5))
        wi, wv = ref.select_by_threshold(acc, s, e, d)
        got = S.select_by_threshold(torch.from_numpy(acc).cuda(), S.PartitionRange(s, e, 0), d)
        assert np.array_equal(got.indices.cpu().numpy(), wi) and np.array_equal(got.values.cpu().numpy(), wv)
        a32 = acc.astype(np.float32)
        oi, ov = o.select(a32, s, e, d)
        g32 = S.select_by_threshold(torch.from_numpy(a32).cuda(), S.PartitionRange(s, e, 0), d)
        assert np.array_equal(g32.indices.cpu().numpy(), oi) and np.array_equal(g32.values.cpu().numpy(), ov)


# test_sparsifier.cpp:154-201 partition-filter invariance and exclusivity
def test_partition_filter_invariance_and_exclusivity():
    rng = np.random.default_rng(17)
    for n in (1, 2, 4, 8):
        for _ in range(20):
            n_g = n + int(rng.integers(0, 50_000))
            acc = torch.from_numpy(rng.standard_normal(n_g)).cuda()
            d = float(rng.uniform(0, 2.5))
            t = int(rng.integers(0, 50))
            whole = S.select_by_threshold(acc, full(acc), d)
            parts = sorted((S.partition(n_g, n, t, i) for i in range(n)), key=lambda r: r.start)
            sels = [S.select_by_threshold(acc, r, d) for r in parts]
            assert torch.equal(torch.cat([s.indices for s in sels]), whole.indices)
            assert torch.equal(torch.cat([s.values for s in sels]), whole.values)
            agg = S.all_gather_indices(sels)
            assert torch.equal(agg.indices, whole.indices)
            assert agg.total_selected() == whole.count() == agg.indices.numel()
            assert S.redundant_traffic_factor(agg) in (0.0, 1.0)


# error_feedback.hpp tests (test_error_feedback.cpp:26-93)
def test_accumulate_compensate_conservation():
    g = vec([3, -1, 2])
    assert torch.equal(S.accumulate(torch.zeros(3, dtype=torch.float64, device="cuda"), 1.0, g), g)
    assert S.accumulate(vec([1, 1]), 0.5, vec([2, 0])).tolist() == [2, 1]
    with pytest.raises(InvalidArgument, match="length mismatch"):
        S.accumulate(vec([1, 1]), 1.0, vec([1, 2, 3]))
    with pytest.raises(InvalidArgument, match="eta must be positive"):
        S.accumulate(vec([1, 1]), 0.0, vec([1, 2]))
    acc = vec([3, 4, 5])
    assert torch.all(S.compensate(acc, [0, 1, 2]) == 0)
    assert torch.equal(S.compensate(acc, []), acc)
    assert S.compensate(acc, [1]).tolist() == [3, 0, 5]
    with pytest.raises(InvalidArgument):
        S.compensate(acc, [7])
    rng = np.random.default_rng(5)
    for _ in range(100):
        n = int(rng.integers(1, 200))
        e = torch.from_numpy(rng.standard_normal(n)).cuda()
        gg = torch.from_numpy(rng.standard_normal(n)).cuda()
        a = S.accumulate(e, 0.05, gg)
        assert torch.equal(a, e + 0.05 * gg)
        sel = torch.from_numpy(np.flatnonzero(rng.integers(0, 3, n) == 0)).cuda()
        sent = torch.zeros_like(a)
        sent[sel] = a[sel]
        assert torch.equal(S.compensate(a, sel) + sent, a)


# test_collectives.cpp:29-101
def test_collectives():
    def sel(ix):
        t = torch.tensor(ix, dtype=torch.int32, device="cuda")
        return S.SparseSelection(t, torch.ones(len(ix), dtype=torch.float64, device="cuda"))
    a = S.all_gather_indices([sel([0, 1]), sel([2, 3])])
    assert a.indices.tolist() == [0, 1, 2, 3] and a.per_worker_counts == [2, 2] and a.total_selected() == 4
    a = S.all_gather_indices([sel([0, 1]), sel([0, 1])])
    assert a.indices.tolist() == [0, 1] and a.total_selected() == 4
    assert S.all_gather_indices([sel([3, 9])]).indices.tolist() == [3, 9]
    accs = [vec([1, 2]), vec([3, 4])]
    assert torch.all(S.all_reduce_sparse(accs, S.AggregatedSelection(torch.empty(0, dtype=torch.int32), [0, 0])) == 0)
    g = S.all_reduce_sparse(accs, S.AggregatedSelection(torch.tensor([1], dtype=torch.int32), [1, 0]))
    assert g.tolist() == [0, 6]
    assert S.all_reduce_sparse([vec([5, -2])], S.AggregatedSelection(torch.tensor([0, 1]), [2])).tolist() == [5, -2]
    with pytest.raises(InvalidArgument):
        S.all_reduce_sparse([vec([1, 2]), vec([1, 2, 3])], S.AggregatedSelection(torch.tensor([1]), [1]))
    rng = np.random.default_rng(23)
    for _ in range(200):
        n = int(rng.integers(1, 5))
        n_g = int(rng.integers(1, 65))
        accs = [torch.from_numpy(rng.standard_normal(n_g)).cuda() for _ in range(n)]
        sels = [sel(np.flatnonzero(rng.integers(0, 4, n_g) == 0).tolist()) for _ in range(n)]
        agg = S.all_gather_indices(sels)
        dense = torch.zeros(n_g, dtype=torch.float64, device="cuda")
        for j in range(n_g):
            for i in range(n):
                dense[j] += accs[i][j]
        masked = torch.zeros_like(dense)
        masked[agg.indices.long()] = dense[agg.indices.long()]
        assert torch.equal(S.all_reduce_sparse(accs, agg), masked)
        assert torch.equal(S.all_reduce_sparse_values(accs, agg), masked[agg.indices.long()])


# error_feedback.hpp:41-48 error_metric (the norm's summation order is not
# pinned by the reference: 1e-12 relative, test_tensor.cpp:57)
@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_error_metric(dtype):
    ref = Reference()
    rng = np.random.default_rng(5)
    for n, n_g in [(1, 1), (1, 3), (2, 1000), (4, 100_003), (3, 2_000_001)]:
        es = [rng.standard_normal(n_g) for _ in range(n)]
        got = S.error_metric([torch.from_numpy(e).to("cuda", dtype) for e in es])
        want = ref.error_metric([e.astype(np.float32).astype(np.float64) if dtype == torch.float32 else e
                                 for e in es])
        assert abs(got - want) <= 1e-12 * want, (n, n_g, got, want)
    assert S.error_metric([torch.zeros(10, dtype=dtype, device="cuda")]) == 0.0
    # deterministic: the same bits every call
    e = torch.randn(3_000_017, dtype=dtype, device="cuda")
    assert len({S.error_metric([e, e]) for _ in range(5)}) == 1
    with pytest.raises(InvalidArgument):
        S.error_metric([])
    with pytest.raises(InvalidArgument):
        S.error_metric([vec([1.0, 2.0]), vec([1.0])])


# test_sparsifier.cpp:71-98 select_topk, sparsifier.cpp:85-108 cltk_select / select_all
@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_select_topk_examples_and_oracle(dtype):
    acc = vec([5, -7, 2, 7], dtype)
    assert S.select_topk(acc, full(acc), 2).indices.tolist() == [1, 3]
    assert S.select_topk(acc, full(acc), 0).count() == 0
    assert S.select_topk(acc, full(acc), 4).indices.tolist() == [0, 1, 2, 3]
    with pytest.raises(InvalidArgument):
        S.select_topk(acc, full(acc), 5)
    tie = vec([2, -2, 2], dtype)
    assert S.select_topk(tie, full(tie), 2).indices.tolist() == [0, 1]
    # zeros among the k largest: the raw acc values come back, sign bits included
    z = vec([0.0, -0.0, 3.0, -0.0, 1.0], dtype)
    got = S.select_topk(z, full(z), 4)
    assert got.indices.tolist() == [0, 1, 2, 4]
    assert torch.signbit(got.values).tolist() == [False, True, False, False]
    rng = np.random.default_rng(7)
    for rep in range(150):
        n = int(rng.integers(1, 401)) if rep < 140 else int(rng.integers(100_000, 300_000))
        a = rng.standard_normal(n)
        if n > 4:
            a[1] = -a[0]
            a[n // 2] = a[0]
        if rep % 3 == 0:
            a = np.round(a * 2) / 2  # many ties
        start = int(rng.integers(0, n)) if rep % 4 == 0 else 0
        k = int(rng.integers(0, n - start + 1))
        t = torch.from_numpy(a).to("cuda", dtype)
        av = np.abs(t.cpu().numpy()[start:]).astype(np.float64)
        order = np.lexsort((np.arange(av.size), -av))[:k] + start  # |acc| desc, index asc
        got = S.select_topk(t, S.PartitionRange(start, n, 0), k)
        assert got.indices.cpu().numpy().tolist() == sorted(order.tolist()), (rep, n, k)
        assert torch.equal(got.values, t[got.indices.long()])


def test_cltk_and_select_all():
    acc = vec([1, -3, 0.5, 2])
    assert S.cltk_select(acc, 1, 1, 5, 4).indices.tolist() == [1]
    with pytest.raises(LogicError):
        S.cltk_select(acc, 1, 0, 5, 4)
    with pytest.raises(InvalidArgument):
        S.cltk_select(acc, 9, 1, 5, 4)
    a = S.select_all(acc)
    assert a.indices.tolist() == [0, 1, 2, 3] and a.values.tolist() == [1, -3, 0.5, 2]


def test_spec_examples_error_metric_accumulate():
    """SPEC.md:200-220 (error_metric, accumulate examples)."""
    assert S.error_metric([torch.zeros(5, dtype=torch.float64, device="cuda")]) == 0.0
    e0 = vec([3.0, 0.0])  # ||e0|| = 3
    e1 = vec([3.0, 4.0])  # ||e1|| = 5
    assert S.error_metric([e0, e1]) == 4.0
    assert S.error_metric([e1]) == 5.0
    g = vec([1.0, 2.0, -0.5])
    e = torch.zeros(3, dtype=torch.float64, device="cuda")
    norms = []
    for _ in range(5):  # no selection, fixed-sign gradient: ||e|| grows monotonically
        e = S.accumulate(e, 0.5, g)
        norms.append(S.error_metric([e]))
    assert all(b > a for a, b in zip(norms, norms[1:]))


@pytest.mark.parametrize("extent,sizes", [(1_000, [7, 300, 0]), (5_000_000, [200_000, 150_000]),
                                          (200_000_000, [400_000, 1, 250_000])])
def test_all_gather_indices_unsorted_overlapping(extent, sizes):
    """collectives.cpp:14-28 is sort + unique of the concatenation for ANY
    input: unsorted, overlapping, duplicated lists — here the bitmap + the
    hand-written popcount scan (scan.cuh) over up to 6M words (several
    passes of the one-CTA tile-total scan)."""
    def sel(ix):
        t = torch.tensor(ix, dtype=torch.int32, device="cuda")
        return S.SparseSelection(t, torch.ones(len(ix), dtype=torch.float64, device="cuda"))
    rng = np.random.default_rng(extent)
    lists = [rng.integers(0, extent, k) for k in sizes]  # unsorted, with duplicates
    lists.append(np.array([extent - 1, 0, extent - 1]))
    agg = S.all_gather_indices([sel(x.tolist()) for x in lists])
    want = np.unique(np.concatenate(lists))
    assert np.array_equal(agg.indices.cpu().numpy().astype(np.int64), want)
    assert agg.per_worker_counts == [len(x) for x in lists]


def test_value_workspace_pool_trim():
    """The value-level calls' scratch comes from a library-owned pool that
    keeps its reserve between calls (micro_value_workspace_trim returns it);
    results are the same before and after a trim."""
    from paper_2310_00967_b200._lib import lib
    acc = torch.randn(300_001, device="cuda") * 0.01
    rng = S.PartitionRange(0, acc.numel(), 0)
    a = S.select_by_threshold(acc, rng, 0.02)
    assert lib().micro_value_workspace_trim(torch.cuda.current_device()) == 0
    b = S.select_by_threshold(acc, rng, 0.02)
    assert torch.equal(a.indices, b.indices) and torch.equal(a.values, b.values)
    assert lib().micro_value_workspace_trim(-1) != 0
