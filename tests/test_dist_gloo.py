"""The multi-rank exchange protocol (paper_2310_00967_b200/dist.exchange) on
CPU over gloo, world size 2 and 3.  The device halves are bound to a numpy
restatement (test-only); every rank's union, sums, residual and threshold
must equal the in-process oracle cluster (harness.cpp:121-224) bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class OracleOps:
    """numpy stand-in for DeviceOps (one rank): the same buffer contract
    (fixed stride kcap, counts in the buffers), CPU tensors."""

    device = torch.device("cpu")
    dtype = torch.float32

    def __init__(self, o, n_g, n, rank, d, delta0, alpha=0.01, eps=1e-12, ef=True):
        self.o, self.n_g, self.n, self.rank = o, n_g, n, rank
        self.e = np.zeros(n_g, np.float32)
        self.delta, self.alpha, self.eps, self.ef = delta0, alpha, eps, ef
        self.k_w = o.per_worker_target_count(d, n_g, n)
        self.kcap = kc = -(-n_g // n)  # the partition size (never overflows)
        self.b = {"own_count": torch.zeros(1, dtype=torch.int64), "own_idx": torch.zeros(kc, dtype=torch.int32),
                  "all_counts": torch.zeros(n, dtype=torch.int64), "all_idx": torch.zeros(n * kc, dtype=torch.int32),
                  "send": torch.zeros(n * kc), "recv": torch.zeros(n * kc), "own_sums": torch.zeros(kc),
                  "all_sums": torch.zeros(n * kc)}

    def buffers(self):
        return self.b

    def compress(self, G, eta, t):
        acc = self.e + np.float32(eta) * G
        s, e = self.o.partition(self.n_g, self.n, t, self.rank)
        self.idx, self.val = self.o.select(acc, s, e, self.delta)
        if self.ef:
            acc[self.idx] = 0
        self.e, self.t = acc, t
        self.b["own_count"][0] = self.idx.size
        self.b["own_idx"][: self.idx.size] = torch.from_numpy(self.idx.astype(np.int32))

    def gather_foreign(self):
        a, cnt, kc = self.b["all_idx"].numpy(), self.b["all_counts"].numpy(), self.kcap
        send = self.b["send"].numpy()
        for o in range(self.n):
            if o == self.rank:
                continue
            j = a[o * kc:o * kc + cnt[o]]
            send[o * kc:o * kc + cnt[o]] = self.e[j]
            if self.ef:
                self.e[j] = 0

    def owner_reduce(self):
        r_, kc = self.b["recv"].numpy(), self.kcap
        k = int(self.b["all_counts"][self.rank])
        s = np.zeros(k, np.float32)
        for r in range(self.n):
            s = s + (self.val if r == self.rank else r_[r * kc:r * kc + k])
        self.b["own_sums"].numpy()[:k] = s

    def finalize(self):
        cnt, kc = self.b["all_counts"].numpy(), self.kcap
        ai, asum = self.b["all_idx"].numpy(), self.b["all_sums"].numpy()
        ui, us = [], []
        for p in range(self.n):
            o = (p - self.t % self.n) % self.n
            ui.append(ai[o * kc:o * kc + cnt[o]])
            us.append(asum[o * kc:o * kc + cnt[o]])
        self.union_idx = np.concatenate(ui)
        self.union_sum = np.concatenate(us)
        self.delta = self.o.update_threshold(self.delta, self.k_w, int(cnt[self.rank]), self.alpha, self.eps)
        if not self.ef:
            self.e[:] = 0


def _worker(rank, world, port, n_g, iters, ef, q):
    import sys
    sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
    from oracle import Oracle, OracleCluster

    from paper_2310_00967_b200.dist import exchange
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    o = Oracle()
    d, delta0, eta = 0.02, 0.015, 0.01
    ops = OracleOps(o, n_g, world, rank, d, delta0, ef=ef)
    ref = OracleCluster(n_g, world, density=d, delta0=delta0, error_feedback=ef)
    bad = []
    for t in range(iters):
        G = np.stack([o.gaussian(3, i, t, n_g) for i in range(world)])
        ops.compress(G[rank], eta, t)
        exchange(ops)
        r = ref.step(G, eta, t)
        if not np.array_equal(ops.union_idx, r["union_idx"]):
            bad.append((t, "union"))
        if not np.array_equal(ops.union_sum, r["union_sum"]):
            bad.append((t, "sums"))
        if not np.array_equal(ops.e, ref.e[rank]):
            bad.append((t, "residual"))
        if ops.delta != r["delta_next"][rank]:
            bad.append((t, "delta"))
    dist.destroy_process_group()
    q.put((rank, bad))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world,n_g,ef", [(2, 10_007, True), (3, 9_001, True), (2, 4_000, False)])
def test_exchange_protocol_gloo(world, n_g, ef):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_g, 12, ef, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, bad in res:
        assert not bad, (rank, bad[:5])
