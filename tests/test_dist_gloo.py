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
    """numpy stand-in for DeviceOps (one rank): same contract, CPU tensors."""

    device = torch.device("cpu")
    dtype = torch.float32
    capacity = 1 << 40

    def __init__(self, o, n_g, n, rank, d, delta0, alpha=0.01, eps=1e-12, ef=True):
        self.o, self.n_g, self.n, self.rank = o, n_g, n, rank
        self.e = np.zeros(n_g, np.float32)
        self.delta, self.alpha, self.eps, self.ef = delta0, alpha, eps, ef
        self.k_w = o.per_worker_target_count(d, n_g, n)

    def compress(self, G, eta, t):
        acc = self.e + np.float32(eta) * G
        s, e = self.o.partition(self.n_g, self.n, t, self.rank)
        self.idx, self.val = self.o.select(acc, s, e, self.delta)
        if self.ef:
            acc[self.idx] = 0
        self.e, self.t = acc, t

    def own_count(self):
        return torch.tensor([self.idx.size], dtype=torch.int64)

    def own_indices(self, kmax):
        out = np.zeros(kmax, np.int32)
        out[: self.idx.size] = self.idx
        return torch.from_numpy(out)

    def gather_foreign(self, all_idx, counts, kmax):
        a = all_idx.numpy()
        parts = []
        for o in range(self.n):
            if o == self.rank:
                continue
            j = a[o * kmax:o * kmax + counts[o]]
            parts.append(self.e[j].copy())
            if self.ef:
                self.e[j] = 0
        return torch.from_numpy(np.concatenate(parts) if parts else np.zeros(0, np.float32))

    def owner_reduce(self, recv, counts, kmax):
        r_ = recv.numpy()
        k = counts[self.rank]
        s = np.zeros(k, np.float32)
        seg = 0
        for r in range(self.n):
            if r == self.rank:
                s = s + self.val
            else:
                s = s + r_[seg:seg + k]
                seg += k
        out = np.zeros(kmax, np.float32)
        out[:k] = s
        return torch.from_numpy(out)

    def finalize(self, all_idx, all_sums, counts, kmax):
        ui, us = [], []
        for p in range(self.n):
            o = (p - self.t % self.n) % self.n
            if kmax:
                ui.append(all_idx.numpy()[o * kmax:o * kmax + counts[o]])
                us.append(all_sums.numpy()[o * kmax:o * kmax + counts[o]])
        self.union_idx = np.concatenate(ui) if ui else np.zeros(0, np.int32)
        self.union_sum = np.concatenate(us) if us else np.zeros(0, np.float32)
        self.delta = self.o.update_threshold(self.delta, self.k_w, counts[self.rank], self.alpha, self.eps)
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
        K = exchange(ops)
        r = ref.step(G, eta, t)
        if K != r["union_idx"].size or not np.array_equal(ops.union_idx, r["union_idx"]):
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
