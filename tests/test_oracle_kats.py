"""Known-answer tests from the reference's own suites, run against BOTH the
C restatement (oracle/micro_oracle.c) and the reference's compiled code
(oracle/_ref).  This pins the oracle before anything is compared with it
(SURVEY.md §8c "KATs and golden vectors to restate").  CPU only."""
import numpy as np
import pytest

from oracle import Oracle, OracleError, Reference


@pytest.fixture(scope="module")
def orc():
    return Oracle()


@pytest.fixture(scope="module")
def ref():
    return Reference()


IMPLS = ["oracle", pytest.param("reference", marks=pytest.mark.ref)]


@pytest.fixture(params=IMPLS)
def impl(request):
    return Oracle() if request.param == "oracle" else Reference()


# test_tensor.cpp:66-71
def test_partition_examples(impl):
    assert impl.partition(8, 4, 0, 2) == (4, 6)
    assert impl.partition(8, 1, 7, 0) == (0, 8)
    assert impl.partition(10, 4, 1, 3) == (0, 3)


# test_tensor.cpp:73-78
@pytest.mark.parametrize("args", [(3, 4, 0, 0), (8, 4, 0, 4), (8, 4, 0, -1), (8, 0, 0, 0), (8, 4, -1, 0)])
def test_partition_rejects(impl, args):
    with pytest.raises(OracleError) as ei:
        impl.partition(*args)
    assert ei.value.code == 1  # invalid_argument


# test_tensor.cpp:80-103 (completeness, disjointness, balance; 300 cases)
def test_partition_property(impl):
    rng = np.random.default_rng(99)
    for _ in range(300):
        n = int(rng.integers(1, 10))
        n_g = n + int(rng.integers(0, 5000))
        t = int(rng.integers(0, 1000))
        rs = sorted(impl.partition(n_g, n, t, i) for i in range(n))
        assert rs[0][0] == 0 and rs[-1][1] == n_g
        lo, hi = n_g // n, n_g // n + (1 if n_g % n else 0)
        for a, b in zip(rs, rs[1:]):
            assert a[1] == b[0]
        for s, e in rs:
            assert lo <= e - s <= hi


# test_tensor.cpp:105-122
def test_partition_cyclic_fairness(impl):
    n_g = 103
    for n in (1, 2, 4, 7):
        allr = {impl.partition(n_g, n, 0, i) for i in range(n)}
        for i in range(n):
            seen = [impl.partition(n_g, n, t, i) for t in range(5, 5 + n)]
            assert len(set(seen)) == n and set(seen) == allr


def _select(impl, acc, s, e, d):
    if isinstance(impl, Reference):
        return impl.select_by_threshold(np.asarray(acc, np.float64), s, e, d)
    return impl.select(np.asarray(acc, np.float64), s, e, d)


# test_sparsifier.cpp:47-61
def test_select_examples(impl):
    acc = [1, -3, 0.5, 2]
    idx, val = _select(impl, acc, 0, 4, 1.5)
    assert idx.tolist() == [1, 3] and val.tolist() == [-3, 2]
    assert _select(impl, acc, 0, 4, 100.0)[0].size == 0
    idx, _ = _select(impl, [0, -0.25, 0, 7], 0, 4, 0.0)
    assert idx.tolist() == [1, 3]


# test_sparsifier.cpp:63-69
def test_select_range(impl):
    idx, _ = _select(impl, [5, 5, 5, 5], 1, 3, 0.0)
    assert idx.tolist() == [1, 2]
    with pytest.raises(OracleError):
        _select(impl, [5, 5, 5, 5], 0, 9, 0.0)
    with pytest.raises(OracleError):
        _select(impl, [5, 5, 5, 5], 0, 4, -1.0)
    with pytest.raises(OracleError):
        _select(impl, [5, 5, 5, 5], 0, 4, float("inf"))


# test_sparsifier.cpp:100-112
def test_threshold_examples(impl):
    assert impl.update_threshold(1.0, 100, 150, 0.1) == pytest.approx(1.1, rel=1e-15)
    assert impl.update_threshold(1.0, 100, 100, 0.1) == 1.0
    assert impl.update_threshold(1.0, 100, 40, 0.1) == pytest.approx(0.9, rel=1e-15)
    assert impl.update_threshold(0.0, 10, 50, 0.1, 1e-12) == 1e-12
    assert impl.update_threshold(0.0, 10, 3, 0.1) == 0.0
    # the exact double the reference produces
    assert impl.update_threshold(1.0, 100, 150, 0.1) == 1.1000000000000001
    for bad in (0.0, 1.0):
        with pytest.raises(OracleError):
            impl.update_threshold(1.0, 10, 5, bad)
    with pytest.raises(OracleError):
        impl.update_threshold(-1.0, 10, 5, 0.5)


# test_sparsifier.cpp:114-129 (sign-correctness, 500 cases)
def test_threshold_sign(impl):
    rng = np.random.default_rng(11)
    for _ in range(500):
        d = float(rng.uniform(1e-9, 10.0))
        a = float(rng.uniform(0.001, 0.999))
        kt, ks = int(rng.integers(0, 1000)), int(rng.integers(0, 1000))
        nx = impl.update_threshold(d, kt, ks, a)
        assert (nx > d) if ks > kt else (nx < d) if ks < kt else (nx == d)
        assert nx >= 0


# test_sparsifier.cpp:217-227
def test_target_counts(impl):
    assert impl.global_target_count(0.01, 10000) == 100
    assert impl.global_target_count(0.001, 100) == 1
    assert impl.global_target_count(1.0, 7) == 7
    for bad in (0.0, 1.5):
        with pytest.raises(OracleError):
            impl.global_target_count(bad, 100)
    assert impl.per_worker_target_count(0.01, 10000, 4) == 25
    assert impl.per_worker_target_count(0.01, 10000, 4, full=True) == 100
    assert impl.per_worker_target_count(0.001, 10000, 16) == 1
    # BASELINE configs
    assert impl.per_worker_target_count(0.01, 11_700_000, 1) == 117_000
    assert impl.per_worker_target_count(0.01, 138_000_000, 8) == 172_500
    assert impl.per_worker_target_count(0.001, 340_000_000, 8) == 42_500


# test_sparsifier.cpp:154-182 (partition-filter invariance) and acceptance.cpp:223-247
def test_partition_filter_invariance(impl):
    rng = np.random.default_rng(13)
    for n in (1, 2, 4, 8):
        for _ in range(40):
            n_g = n + int(rng.integers(0, 2000))
            acc = rng.standard_normal(n_g)
            d = float(rng.uniform(0, 2.5))
            t = int(rng.integers(0, 50))
            whole_i, whole_v = _select(impl, acc, 0, n_g, d)
            parts = sorted((impl.partition(n_g, n, t, i) for i in range(n)))
            mi = np.concatenate([_select(impl, acc, s, e, d)[0] for s, e in parts])
            mv = np.concatenate([_select(impl, acc, s, e, d)[1] for s, e in parts])
            assert np.array_equal(mi, whole_i) and np.array_equal(mv, whole_v)


def test_oracle_f32_select_matches_double_predicate(orc):
    """The f32 contract: (double)|acc_f32| > delta, i.e. |acc| > rd_f32(delta)."""
    rng = np.random.default_rng(5)
    acc = rng.standard_normal(20000).astype(np.float32)
    for d in (0.0, 0.5, 1.0, 1.0000000001, float(np.float32(1.7)), 2.575829303548901):
        idx, val = orc.select(acc, 0, acc.size, d)
        want = np.flatnonzero(np.abs(acc).astype(np.float64) > d)
        assert np.array_equal(idx, want) and np.array_equal(val, acc[want])


# test_error_feedback.cpp:26-32, 46-65, 67-93 (reference side)
@pytest.mark.ref
def test_accumulate_compensate(ref):
    g = np.array([3, -1, 2.0])
    assert np.array_equal(ref.accumulate(np.zeros(3), 1.0, g), g)
    assert ref.accumulate(np.array([1, 1.0]), 0.5, np.array([2, 0.0])).tolist() == [2, 1]
    with pytest.raises(OracleError):
        ref.accumulate(np.array([1, 1.0]), 1.0, np.array([1, 2, 3.0]))
    with pytest.raises(OracleError):
        ref.accumulate(np.array([1, 1.0]), 0.0, np.array([1, 2.0]))
    acc = np.array([3, 4, 5.0])
    assert np.all(ref.compensate(acc, [0, 1, 2]) == 0)
    assert np.array_equal(ref.compensate(acc, []), acc)
    assert ref.compensate(acc, [1]).tolist() == [3, 0, 5]
    with pytest.raises(OracleError):
        ref.compensate(acc, [7])


# test_collectives.cpp:29-66
@pytest.mark.ref
def test_collectives_examples(ref):
    u, c, tot = ref.all_gather_indices([[0, 1], [2, 3]])
    assert u.tolist() == [0, 1, 2, 3] and c.tolist() == [2, 2] and tot == 4
    u, c, tot = ref.all_gather_indices([[0, 1], [0, 1]])
    assert u.tolist() == [0, 1] and tot == 4
    accs = np.array([[1, 2], [3, 4.0]])
    assert np.all(ref.all_reduce_sparse(accs, []) == 0)
    assert ref.all_reduce_sparse(accs, [1]).tolist() == [0, 6]
    assert ref.all_reduce_sparse(np.array([[5, -2.0]]), [0, 1]).tolist() == [5, -2]


# test_collectives.cpp:68-101: worker-order dense sum then mask, bitwise (200 cases)
@pytest.mark.ref
def test_all_reduce_equals_dense_then_mask(ref, orc):
    rng = np.random.default_rng(23)
    for _ in range(200):
        n = int(rng.integers(1, 5))
        n_g = int(rng.integers(1, 65))
        accs = rng.standard_normal((n, n_g))
        sels = [np.flatnonzero(rng.integers(0, 4, n_g) == 0) for _ in range(n)]
        u, _, _ = ref.all_gather_indices(sels)
        dense = np.zeros(n_g)
        for j in range(n_g):
            for i in range(n):
                dense[j] += accs[i, j]
        got = ref.all_reduce_sparse_values(accs, u)
        assert np.array_equal(got, dense[u])
        assert np.array_equal(orc.all_reduce_sparse_values(accs, u), dense[u])
        f = accs.astype(np.float32)
        d32 = np.zeros(n_g, np.float32)
        for i in range(n):
            d32 = d32 + f[i]
        assert np.array_equal(orc.all_reduce_sparse_values(f, u), d32[u])


def test_learning_rate_schedule():
    """harness.cpp:61-63, 109-110 (host arithmetic of the Python face)."""
    from paper_2310_00967_b200.sparsim import LrSchedule, learning_rate_at, resolve_decay_at
    lr = LrSchedule(initial=0.1, decay_factor=0.5, decay_at=-1)
    assert resolve_decay_at(lr, 200) == 150
    assert learning_rate_at(lr, 150, 149) == 0.1 and learning_rate_at(lr, 150, 150) == 0.05
    assert resolve_decay_at(LrSchedule(decay_at=7), 200) == 7


def test_kind_names():
    """sparsifier.cpp:136-160."""
    from paper_2310_00967_b200._lib import InvalidArgument
    from paper_2310_00967_b200.sparsim import parse_per_worker_target, parse_sparsifier_kind
    assert parse_sparsifier_kind("hard_threshold") == "hard" and parse_sparsifier_kind("topk") == "topk"
    assert parse_per_worker_target("full") == "full"
    with pytest.raises(InvalidArgument):
        parse_sparsifier_kind("foo")
    with pytest.raises(InvalidArgument):
        parse_per_worker_target("half")
