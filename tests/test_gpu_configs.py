"""Every BASELINE.json config at its full size, bit-exact against the oracle
every iteration (GPU only).

The reference defines the path over whole runs (run_iteration,
harness.cpp:121-224; acceptance runs of 2000 iterations,
acceptance.cpp:93-118, :174-220).  These tests run the CUDA path and the
checker side by side on the same synthetic gradients at the sizes BASELINE
quotes and compare, at every iteration: per-worker counts, the union
(indices and sums), the next thresholds (exact doubles, not 1e-6), and —
at the checkpoints named per test — every worker's residual, the model and
the dense g/n.

  C1  11.7M, d = 0.01, n = 1: the 100 adaptation iterations from the
      reference's default delta_0 = 0.01, fp32 (restatement) and fp64 (the
      reference's own compiled code); the threshold trajectory over 1000.
  C2  11.7M, n = 2/4/8: the in-process cluster and GroupMicro (one context
      per rank, the peer exchange), 20 iterations.
  C3  138M, n = 8: cluster and GroupMicro, 3 iterations.
  C4  340M, d = 0.001, n = 1: 3 iterations.
  C5  1.5B, d = 0.001 / 0.01 / 0.1, n = 1: 2 iterations each (at d = 0.1
      150M pairs per step, indices up to 70 % of int32).

Gradients: include/micro_synth.h generated on the device (bit-identical to
the host generator: test_gpu_parity.py) and copied to the host for the
checker.
"""
import gc
import statistics

import numpy as np
import pytest
import torch

from oracle import OracleCluster, RefCluster

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2310_00967_b200 import engine
    from paper_2310_00967_b200.dist import GroupMicro

ETA, ALPHA, SEED = 0.01, 0.01, 1


def warm_delta0(d):
    """The 1 - d quantile of |eta G|, G ~ N(0, 1) (SURVEY.md 8d warm start)."""
    return statistics.NormalDist().inv_cdf(1 - d / 2) * ETA


def grads(n, n_g, t, dtype, buf):
    """Device gradients of the n workers at iteration t (one fresh stream per
    (worker, t)) and their host copy for the checker."""
    out = []
    for i in range(n):
        engine.synth_gaussian(buf[i], SEED, i, t)
        out.append(buf[i])
    host = np.stack([b.cpu().numpy() for b in out]).astype(dtype)
    dev = [torch.from_numpy(host[i]).cuda() for i in range(n)] if dtype == np.float64 else out
    return dev, host


def check_step(m, r, t, tag=""):
    st = m.query()
    idx, sums = m.union()
    assert st.K == r["union_idx"].size, (tag, t, "K", st.K, r["union_idx"].size)
    assert np.array_equal(idx.astype(np.int64), r["union_idx"]), (tag, t, "union")
    assert np.array_equal(sums, r["union_sum"].astype(sums.dtype)), (tag, t, "sums")
    return st


class Run:
    """The CUDA path (a single-device cluster, optionally also GroupMicro) and
    the checker (restatement or the reference's code) stepped together."""

    def __init__(self, n_g, n, d, delta0, dtype=np.float32, checker="restatement", group=False, dense=True,
                 grad32=False):
        self.n_g, self.n, self.d = n_g, n, d
        self.dtype = dtype
        self.grad32 = grad32  # fp32 gradients into the fp64 engine (micro_config.grad_dtype)
        tdt = torch.float32 if dtype == np.float32 else torch.float64
        self.m = engine.Micro(n_g, n, dtype=tdt, density=d, initial_threshold=delta0, scaling_factor=ALPHA,
                              dense_output=dense, grad_dtype=torch.float32 if grad32 else tdt)
        self.x = torch.zeros(n_g, dtype=tdt, device="cuda")
        self.m.set_model(self.x)
        self.g = None
        if group:
            self.g = GroupMicro(n_g, n, devices=[0] * n, dtype=tdt, density=d, initial_threshold=delta0,
                                scaling_factor=ALPHA, dense_output=False)
            self.gx = [torch.zeros(n_g, dtype=tdt, device="cuda") for _ in range(n)]
            for rm, x in zip(self.g.ranks, self.gx):
                rm.set_model(x)
        if checker == "reference":
            self.ref = RefCluster(n_g, n, d, delta0, ALPHA, 1e-12, False, True, model=True)
        else:
            self.ref = OracleCluster(n_g, n, d, delta0, ALPHA, 1e-12, False, True, dtype=dtype, model=True)
        self.checker = checker
        self.buf = [torch.empty(n_g, device="cuda") for _ in range(n)]

    def residuals(self):
        return self.ref.residuals() if self.checker == "reference" else self.ref.e

    def step(self, t, full_check=False):
        if self.grad32:  # the device keeps fp32; the checker gets the same values widened (exact)
            dev, host = grads(self.n, self.n_g, t, np.float32, self.buf)
            host = host.astype(np.float64)
        else:
            dev, host = grads(self.n, self.n_g, t, self.dtype, self.buf)
        torch.cuda.synchronize()
        self.m.step(dev, ETA, t)
        if self.g is not None:
            self.g.step(dev, ETA, t)
        r = self.ref.step(host, ETA, t)
        st = check_step(self.m, r, t, "cluster")
        assert np.array_equal(st.counts, r["counts"]), (t, "counts")
        assert np.array_equal(st.deltas, r["delta_next"]), (t, "delta", st.deltas, r["delta_next"])
        if self.g is not None:
            self.g.synchronize()
            for rank, rm in enumerate(self.g.ranks):
                rst = check_step(rm, r, t, f"group rank {rank}")
                assert rst.counts[0] == r["counts"][rank], (t, rank, "count")
                assert rst.deltas[0] == r["delta_next"][rank], (t, rank, "delta")
        if full_check:
            self.check_state(t, r)
        return r

    def check_state(self, t, r):
        want = self.residuals()
        for i in range(self.n):
            assert np.array_equal(self.m.residual(i), want[i].astype(self.dtype)), (t, "residual", i)
        xw = self.ref.x.astype(self.dtype)
        assert np.array_equal(self.x.cpu().numpy(), xw), (t, "model")
        dense = self.m.dense()
        dw = np.zeros(self.n_g, self.dtype)
        dw[r["union_idx"]] = (r["union_sum"].astype(self.dtype) / self.dtype(self.n))
        assert np.array_equal(dense, dw), (t, "dense g/n")
        if self.g is not None:
            for rank, rm in enumerate(self.g.ranks):
                assert np.array_equal(rm.residual(0), want[rank].astype(self.dtype)), (t, "group residual", rank)
                assert np.array_equal(self.gx[rank].cpu().numpy(), xw), (t, "group model", rank)

    def close(self):
        self.m.close()
        if self.g is not None:
            self.g.close()
        del self.ref, self.buf, self.x
        gc.collect()
        torch.cuda.empty_cache()


def test_c1_adaptation_f32_and_threshold_trajectory():
    """C1: 11.7M, d = 0.01, n = 1 from the reference's default delta_0 = 0.01
    (sparsifier.hpp:42; 32 % selected at t = 0).  Bit-exact every iteration
    for the 100 adaptation iterations (state checked at t = 0, 1, 49, 99),
    then the threshold trajectory delta_t compared exactly (and counts every
    iteration, the union every 25th) through t = 999."""
    run = Run(11_700_000, 1, 0.01, 0.01)
    for t in range(1000):
        if t < 100 or t % 25 == 0 or t == 999:
            run.step(t, full_check=t in (0, 1, 49, 99, 999))
        else:  # counts and thresholds only (no union copy)
            dev, host = grads(1, run.n_g, t, np.float32, run.buf)
            run.m.step(dev, ETA, t)
            r = run.ref.step(host, ETA, t)
            st = run.m.query()
            assert st.counts[0] == r["counts"][0], (t, "count")
            assert st.deltas[0] == r["delta_next"][0], (t, "delta")
    h = run.m.history(1000)
    assert h["t"].tolist() == list(range(1000))
    run.close()


def test_c1_adaptation_f64_reference_code():
    """C1 in the reference's own arithmetic: 100 iterations against its
    compiled sparsifier/collectives code (oracle/_ref), bit for bit."""
    run = Run(11_700_000, 1, 0.01, 0.01, dtype=np.float64, checker="reference")
    for t in range(100):
        run.step(t, full_check=t in (0, 1, 50, 99))
    run.close()


def test_c1_fp32_gradients_f64_reference_code():
    """C1 as BASELINE states it ("fp32 gradient") in the reference's fp64
    arithmetic: fp32 gradients into the f64 engine, 100 iterations against
    the reference's compiled code fed the same values, bit for bit."""
    run = Run(11_700_000, 1, 0.01, 0.01, dtype=np.float64, checker="reference", grad32=True)
    for t in range(100):
        run.step(t, full_check=t in (0, 1, 50, 99))
    run.close()


def test_c3_fp32_gradients_f64_n1():
    """The bench's default step (C3's per-GPU slice: 138M, d = 0.01, n = 1,
    fp32 gradients, fp64 state and arithmetic, model + dense g/n) against
    the reference's own code, 3 iterations from the warm delta_0."""
    run = Run(138_000_000, 1, 0.01, warm_delta0(0.01), dtype=np.float64, checker="reference", grad32=True)
    for t in range(3):
        run.step(t, full_check=t == 2)
    run.close()


@pytest.mark.parametrize("n", [2, 4, 8])
def test_c2_partitioned_cluster_and_group(n):
    """C2: 11.7M over n = 2/4/8 workers — the in-process cluster and the n-rank
    peer exchange (GroupMicro, all ranks on cuda:0) — 20 iterations."""
    run = Run(11_700_000, n, 0.01, warm_delta0(0.01), group=True)
    for t in range(20):
        run.step(t, full_check=t in (0, 9, 19))
    run.close()


def test_c3_vgg16_n8():
    """C3: 138M, d = 0.01, n = 8, error feedback on: the cluster and the 8-rank
    peer exchange, 3 iterations."""
    run = Run(138_000_000, 8, 0.01, warm_delta0(0.01), group=True)
    for t in range(3):
        run.step(t, full_check=t == 2)
    run.close()


def test_c4_bert_large_n1():
    """C4: 340M, d = 0.001, n = 1, 3 iterations."""
    run = Run(340_000_000, 1, 0.001, warm_delta0(0.001))
    for t in range(3):
        run.step(t, full_check=t == 2)
    run.close()


@pytest.mark.parametrize("d", [0.001, 0.01, 0.1])
def test_c5_gpt2xl_density_sweep(d):
    """C5: 1.5B, n = 1, d = 0.001 / 0.01 / 0.1, 2 iterations each.  At d = 0.1
    a step selects ~150M pairs: k1_gather's super-block offsets (1024 super
    blocks of many runs) and int32 indices up to 1.5e9 are all exercised."""
    run = Run(1_500_000_000, 1, d, warm_delta0(d))
    for t in range(2):
        r = run.step(t, full_check=t == 1)
    assert r["union_idx"][-1] > 1_000_000_000
    run.close()
