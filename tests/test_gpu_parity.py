"""Parity of the CUDA path (through the C ABI) with the oracle — GPU only.

Chain of trust, link 2: GPU fp32 == C restatement fp32, and GPU fp64 == the
reference's own compiled code (oracle/_ref) and its golden runs, BIT FOR BIT:
per-worker counts, union indices, reduced sums, thresholds, residuals, the
dense averaged gradient and the model.
"""
import functools
import glob
import operator
import os

import numpy as np
import pytest
import torch

from oracle import Oracle, OracleCluster, RefCluster

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2310_00967_b200 import engine
    from paper_2310_00967_b200._lib import (CapacityError, InvalidArgument, LogicError,
                                            NonFiniteGradient)

SEED, ETA = 7, 0.01


def seq_sum(xs):
    """Left-to-right fp64 sum (the reference's loops; numpy and Python's sum() are not)."""
    return functools.reduce(operator.add, (float(x) for x in xs), 0.0)


def gen(o, n, n_g, t, dtype):
    return np.stack([o.gaussian(SEED, i, t, n_g) for i in range(n)]).astype(dtype)


def run_pair(n_g, n, d, delta0, iters, dtype=np.float32, full=False, ef=True, oracle="restatement",
             check_every=1, split=False, unaligned=False, grad32=False, alpha=0.01):
    """grad32: fp32 gradients into the fp64 engine (micro_config.grad_dtype);
    the checker runs fp64 on the same values widened."""
    o = Oracle()
    tdt = torch.float32 if dtype == np.float32 else torch.float64
    assert not grad32 or dtype == np.float64
    gdt = torch.float32 if grad32 else tdt
    m = engine.Micro(n_g, n, dtype=tdt, density=d, initial_threshold=delta0, target="full" if full else "split",
                     error_feedback=ef, grad_dtype=gdt, scaling_factor=alpha)
    x = torch.zeros(n_g, dtype=tdt, device="cuda")
    m.set_model(x)
    if oracle == "reference":
        ref = RefCluster(n_g, n, d, delta0, alpha, 1e-12, full, ef, model=True)
    else:
        ref = OracleCluster(n_g, n, d, delta0, alpha, 1e-12, full, ef, dtype=dtype, model=True)
    recs_want = []  # per step: (K, sum k_i, threshold used, error norm) from the checker
    for t in range(iters):
        thr_used = seq_sum(m.query().deltas) / n
        G = gen(o, n, n_g, t, dtype)
        G32 = None
        if grad32:
            G32 = gen(o, n, n_g, t, np.float32)
            G = G32.astype(np.float64)  # exact
        # energy before the exchange zeroes foreign entries: at n > 1 the
        # norm is ||e||^2 - (squares zeroed by the exchange), accurate to
        # ~1e-15 of this, not of the result
        e_now = ref.residuals() if oracle == "reference" else ref.e
        acc = e_now.astype(dtype) + dtype(ETA) * G
        energy = float(np.sqrt((acc.astype(np.float64) ** 2).sum(axis=1)).max())
        Gd = list(torch.from_numpy(G32 if grad32 else G).cuda())
        if unaligned:  # gradients off the 16-byte grid: the library realigns them (staging copy)
            buf = torch.empty((n, n_g + 1), dtype=gdt, device="cuda")
            buf[:, 1:] = torch.stack(Gd)
            Gd = [buf[i, 1:] for i in range(n)]
            assert Gd[0].data_ptr() % 16
        if split:  # micro_compress + micro_aggregate (k_finalize launched separately)
            m.compress(Gd, ETA, t)
            m.aggregate()
        else:      # micro_step (n = 1: threshold update folded into k1_gather)
            m.step(Gd, ETA, t)
        r = ref.step(G, ETA, t)
        E = ref.residuals() if oracle == "reference" else ref.e
        norms = np.sqrt((E.astype(np.float64) ** 2).sum(axis=1))
        recs_want.append((r["union_idx"].size, int(np.sum(r["counts"])), thr_used, seq_sum(norms) / n, energy))
        if t % check_every and t != iters - 1:
            continue
        st = m.query()
        idx, sums = m.union()
        assert np.array_equal(st.counts, r["counts"]), t
        assert st.K == r["union_idx"].size, t
        assert np.array_equal(idx.astype(np.int64), r["union_idx"]), t
        assert np.array_equal(sums, r["union_sum"].astype(sums.dtype)), t
        assert np.array_equal(st.deltas, r["delta_next"]), t
        res = np.stack([m.residual(i) for i in range(n)])
        want = ref.residuals() if oracle == "reference" else ref.e
        assert np.array_equal(res, want.astype(res.dtype)), t
        dense = m.dense()
        dw = np.zeros(n_g, dense.dtype)
        dw[r["union_idx"]] = (r["union_sum"] / n).astype(dense.dtype) if dtype == np.float64 else \
            (r["union_sum"].astype(np.float32) / np.float32(n))
        assert np.array_equal(dense, dw), t
        assert np.array_equal(x.cpu().numpy(), ref.x.astype(dense.dtype)), t
    h = m.history(iters)
    assert h["t"].tolist() == list(range(iters))
    k_glob = Oracle().global_target_count(d, n_g)
    for t, (rec, (K, tot, thr, en, energy)) in enumerate(zip(m.records(iters), recs_want)):
        # the reference's IterationRecord (harness.cpp:226-236)
        assert rec["t"] == t and rec["K"] == K and rec["total_selected"] == tot
        assert rec["actual_density"] == K / n_g
        assert rec["buildup_factor"] == (K / k_glob if tot else 0.0)
        assert rec["redundant_traffic_factor"] == (tot / K if tot else 0.0)
        assert rec["threshold"] == thr
        if n == 1 or en > 1e-6 * energy:
            assert abs(rec["error_norm"] - en) <= 1e-12 * en + 1e-300, (t, rec["error_norm"], en)
        else:  # (nearly) everything zeroed: the subtraction's noise floor
            assert rec["error_norm"] <= 1e-6 * energy, (t, rec["error_norm"], en, energy)
    m.close()


@pytest.mark.parametrize("n_g,n,d,delta0,oracle", [
    (100_003, 1, 0.01, 0.02, "reference"),
    (65_537, 4, 0.02, 0.01, "reference"),
    (20_000, 3, 0.05, 0.01, "restatement"),
    (4_095, 1, 0.3, 0.5, "reference"),     # one partial unit
])
def test_gpu_fp32_gradients_fp64_state(n_g, n, d, delta0, oracle, k1_kernel):
    """BASELINE's "fp32 gradient" in the reference's fp64 arithmetic
    (micro_config.grad_dtype = MICRO_GRAD_F32): bit-exact with the reference's
    own code (and the fp64 restatement) fed the same gradient values widened
    to double — counts, union, sums, thresholds, residuals, dense g/n, model."""
    run_pair(n_g, n, d, delta0, iters=12, dtype=np.float64, oracle=oracle, grad32=True, unaligned=k1_kernel)


@pytest.mark.parametrize("alpha", [0.003, 0.001, 0.3])
def test_gpu_controller_alpha(alpha):
    """The bench's alpha (0.003) and others: the controller is the same code
    path, bit-exact with the reference's own code (fp64 on fp32 gradients)."""
    run_pair(65_537, 1, 0.01, 0.02, iters=30, dtype=np.float64, oracle="reference", grad32=True, alpha=alpha)
    run_pair(20_011, 3, 0.02, 0.01, iters=15, alpha=alpha)


@pytest.fixture(params=["aligned", "unaligned"])
def k1_kernel(request):
    """Gradient placement: 16-byte aligned (K1 streams it directly) or not
    (the library realigns it into its staging buffer first)."""
    return request.param == "unaligned"


@pytest.mark.parametrize("n_g,n,d,delta0", [
    (10_000, 1, 0.01, 0.01),
    (10_007, 2, 0.01, 0.02),
    (9_999, 3, 0.05, 0.01),
    (65_537, 4, 0.01, 0.025),
    (100_003, 8, 0.02, 0.01),
    (4_096, 16, 0.01, 0.01),
    (5, 5, 0.5, 0.0),          # n_g == n: one element per partition
    (4_095, 1, 0.3, 0.5),      # one partial tile
    (123_457, 7, 0.001, 0.03),
])
def test_gpu_f32_matches_restatement(n_g, n, d, delta0, k1_kernel):
    run_pair(n_g, n, d, delta0, iters=25, unaligned=k1_kernel)


@pytest.mark.parametrize("full,ef", [(True, True), (False, False), (True, False)])
def test_gpu_f32_modes(full, ef, k1_kernel):
    run_pair(20_000, 4, 0.01, 0.01, iters=15, full=full, ef=ef, unaligned=k1_kernel)
    run_pair(20_000, 1, 0.01, 0.01, iters=15, full=full, ef=ef, unaligned=k1_kernel)


@pytest.mark.parametrize("n_g,n", [(10_000, 1), (65_537, 1), (10_007, 2)])
def test_gpu_split_compress_aggregate(n_g, n):
    """The two-call API and the single micro_step give the same iteration."""
    run_pair(n_g, n, 0.01, 0.01, iters=12, split=True)
    run_pair(n_g, n, 0.01, 0.01, iters=12, dtype=np.float64, split=True)


@pytest.mark.parametrize("n_g,n", [(5_000_011, 1), (5_000_011, 3), (40_000_003, 1)])
def test_gpu_many_super_blocks(n_g, n):
    """k1_gather's offsets over many super blocks (40M: super blocks of > 8 runs)."""
    run_pair(n_g, n, 0.01, 0.03, iters=3)


def test_gpu_density_one_threshold_zero():
    """test_harness.cpp:60-76: d = 1, delta0 = 0 -> everything nonzero is sent."""
    run_pair(8_192, 4, 1.0, 0.0, iters=8)


@pytest.mark.ref
@pytest.mark.parametrize("n_g,n,d,delta0", [(10_000, 1, 0.01, 0.01), (10_007, 2, 0.01, 0.02),
                                             (12_345, 8, 0.02, 0.01), (3_001, 3, 0.1, 0.05)])
def test_gpu_f64_matches_reference_code(n_g, n, d, delta0, k1_kernel):
    run_pair(n_g, n, d, delta0, iters=20, dtype=np.float64, oracle="reference", unaligned=k1_kernel)


GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "micro_ref64_*.npz")))


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p)[12:-4] for p in GOLDEN])
def test_gpu_f64_reproduces_golden(path):
    z = np.load(path)
    n_g, n, d, delta0, full, ef, iters, seed, eta = z["config"].tolist()
    n_g, n, iters, seed = int(n_g), int(n), int(iters), int(seed)
    o = Oracle()
    m = engine.Micro(n_g, n, dtype=torch.float64, density=d, initial_threshold=delta0,
                     target="full" if full else "split", error_feedback=bool(ef))
    x = torch.zeros(n_g, dtype=torch.float64, device="cuda")
    m.set_model(x)
    off = 0
    for t in range(iters):
        G = torch.from_numpy(np.stack([o.gaussian(seed, i, t, n_g) for i in range(n)]).astype(np.float64)).cuda()
        m.step(list(G), eta, t)
        K = int(z["K"][t])
        st = m.query()
        idx, sums = m.union()
        assert np.array_equal(st.counts, z["counts"][t])
        assert np.array_equal(idx, z["union_idx"][off:off + K])
        assert np.array_equal(sums, z["union_sum"][off:off + K])
        assert np.array_equal(st.deltas, z["delta_next"][t])
        off += K
    assert np.array_equal(np.stack([m.residual(i) for i in range(n)]), z["residuals"])
    assert np.array_equal(x.cpu().numpy(), z["model"])


def test_synthetic_gradients_bit_identical_host_device():
    o = Oracle()
    for n, w, t in [(1_000_003, 0, 0), (4097, 3, 11), (7, 1, 2**33)]:
        g = torch.empty(n, device="cuda")
        engine.synth_gaussian(g, SEED, w, t)
        assert np.array_equal(g.cpu().numpy().view(np.uint32), o.gaussian(SEED, w, t, n).view(np.uint32))


def test_nonfinite_gradient_poisons_until_reset():
    m = engine.Micro(10_000, 2)
    G = torch.randn(2, 10_000, device="cuda")
    G[1, 1234] = float("nan")
    m.step(list(G), ETA, 0)
    with pytest.raises(NonFiniteGradient, match="non-finite gradient"):
        m.sync()
    with pytest.raises(NonFiniteGradient):
        m.step(list(torch.randn(2, 10_000, device="cuda")), ETA, 1)
    m.reset()
    m.step(list(torch.randn(2, 10_000, device="cuda")), ETA, 0)
    m.sync()
    G = torch.randn(1, 10_000, device="cuda")
    G[0, 5] = float("inf")
    m1 = engine.Micro(10_000, 1)
    m1.step(list(G), ETA, 0)
    with pytest.raises(NonFiniteGradient):
        m1.sync()


def test_capacity_overflow_reported():
    m = engine.Micro(50_000, 1, selection_capacity=100, initial_threshold=0.0)
    m.step([torch.randn(50_000, device="cuda")], ETA, 0)
    with pytest.raises(CapacityError):
        m.sync()


def test_config_rejections():
    with pytest.raises(InvalidArgument):
        engine.Micro(3, 4)
    with pytest.raises(InvalidArgument):
        engine.Micro(100, 2, density=0.0)
    with pytest.raises(InvalidArgument):
        engine.Micro(100, 2, scaling_factor=1.0)
    with pytest.raises(InvalidArgument):
        engine.Micro(100, 2, initial_threshold=-1.0)
    with pytest.raises(InvalidArgument):
        engine.Micro(100, 2, min_threshold=0.0)
    m = engine.Micro(100, 1)
    with pytest.raises(InvalidArgument):
        m.step([torch.randn(100, device="cuda")], 0.0, 0)   # eta must be positive
    with pytest.raises(InvalidArgument):
        m.step([torch.randn(100, device="cuda")], ETA, -1)  # negative iteration
    with pytest.raises(LogicError):
        m.aggregate()                                       # without compress


def test_step_host_end_to_end():
    o = Oracle()
    n_g = 50_001
    m = engine.Micro(n_g, 2)
    ref = OracleCluster(n_g, 2)
    for t in range(5):
        G = gen(o, 2, n_g, t, np.float32)
        h = torch.from_numpy(G).pin_memory()
        idx, sums = m.step_host(h, ETA, t)
        r = ref.step(G, ETA, t)
        assert np.array_equal(idx, r["union_idx"]) and np.array_equal(sums, r["union_sum"])


def test_full_size_properties_138M():
    """BASELINE C3 size at n = 1: size-independent properties — ordered unique indices inside the partition, |acc| > delta,
    conservation e_{t+1} + sent == e_t + eta*G elementwise, count == the
    torch-computed count, dense == sums at the union."""
    n_g = 138_000_000
    torch.cuda.empty_cache()
    m = engine.Micro(n_g, 1, initial_threshold=2.576 * ETA)
    G = torch.empty(n_g, device="cuda")
    for t in range(3):
        engine.synth_gaussian(G, SEED, 0, t)
        e0 = m.residual_device(0).clone()
        m.step([G], ETA, t)
        st = m.query()
        delta = m.history(1)["delta_used"][0, 0]
        acc = e0 + torch.tensor(ETA, dtype=torch.float32) * G
        sel = acc.abs().double() > delta
        assert int(sel.sum()) == st.K
        idx, sums = m.union()
        it = torch.from_numpy(idx.astype(np.int64)).cuda()
        assert torch.equal(it, torch.nonzero(sel).flatten())
        assert torch.equal(torch.from_numpy(sums).cuda(), acc[it])
        e1 = m.residual_device(0)
        sent = torch.zeros_like(acc)
        sent[it] = acc[it]
        assert torch.equal(e1 + sent, acc)
        dense = m.dense_device()
        assert torch.equal(dense[it], acc[it]) and int((dense != 0).sum()) == st.K
        del e0, acc, sel, sent
    m.close()
    torch.cuda.empty_cache()


def test_gpu_records_to_reference_format(tmp_path):
    """§8f-2: a GPU run's records written in the reference's CSV/JSON format
    (report.py, byte-identical to report.cpp — tests/test_report.py) and read back."""
    from paper_2310_00967_b200 import report
    o = Oracle()
    m = engine.Micro(50_000, 2, density=0.01, initial_threshold=0.02)
    for t in range(6):
        m.step(list(torch.from_numpy(gen(o, 2, 50_000, t, np.float32)).cuda()), ETA, t)
    recs = m.records()
    cfg = report.config_for(m, lr=ETA, iterations=6, seed=SEED)
    for fmt in ("csv", "json"):
        p = tmp_path / f"run.{fmt}"
        report.emit(cfg, recs, fmt, str(p))
        assert p.read_text().count("\n") > 6
    back = report.read_records_json(str(tmp_path / "run.json"))
    assert [r["error_norm"] for r in back["records"]] == [r["error_norm"] for r in recs]
    assert back["config"]["workers"] == 2 and back["config"]["density"] == 0.01
    m.close()


@pytest.mark.parametrize("n_g,grad32", [(1_000_003, False), (65_536 * 3 + 17, False), (1_000_003, True)])
def test_gpu_step_host_pipelined_matches_device_step(n_g, grad32):
    """micro_step_host (gradient copied in chunks on a copy stream, K1
    streaming each chunk as it lands) == micro_step on device gradients;
    grad32: fp32 host gradients into the fp64 engine (half the PCIe bytes)."""
    o = Oracle()
    kw = dict(dtype=torch.float64, grad_dtype=torch.float32) if grad32 else {}
    a = engine.Micro(n_g, 1, density=0.01, initial_threshold=0.02, **kw)
    b = engine.Micro(n_g, 1, density=0.01, initial_threshold=0.02, **kw)
    xdt = torch.float64 if grad32 else torch.float32
    xa = torch.zeros(n_g, device="cuda", dtype=xdt)
    xb = torch.zeros(n_g, device="cuda", dtype=xdt)
    a.set_model(xa)
    b.set_model(xb)
    for t in range(6):
        G = o.gaussian(SEED, 0, t, n_g)
        hG = torch.from_numpy(G).pin_memory()
        ia, sa = a.step_host(hG, ETA, t)
        b.step([torch.from_numpy(G).cuda()], ETA, t)
        ib, sb = b.union()
        assert np.array_equal(ia, ib) and np.array_equal(sa, sb), t
        assert np.array_equal(a.residual(0), b.residual(0)), t
        assert torch.equal(xa, xb), t
    a.close()
    b.close()
