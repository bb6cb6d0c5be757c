"""One process per GPU: the MiCRO exchange over torch.distributed (NCCL).

Each rank is one worker i of the n-worker cluster.  Per iteration
(reference semantics collectives.cpp:14-57, harness.cpp:185-224):

  K1   micro_compress: acc_i = e_i + eta*G_i, own selection S_i (partition
       (t % n + i) % n), own residual entries zeroed          [device]
  K2   all-gather k_i                                          [NCCL]
  K3   all-gather S_i indices, padded to kmax = max_i k_i      [NCCL]
  K4   gather acc_i at every other owner's indices, zero them  [device]
  K5   all-to-all-v: contributions -> their owners             [NCCL]
  K6   owner: s = 0; s += contribution_r for r = 0..n-1        [device]
  K7   all-gather the owners' sums, padded to kmax             [NCCL]
  K8   union in partition order, dense g/n, model, delta_i     [device]

The partitions are exclusive, so the union restricted to partition p is the
selection of p's owner: no sort, no build-up, and every sum is formed in
worker order from +0 exactly like all_reduce_sparse_values.  `ncclAllReduce`
is never used: its reduction order is not the reference's.

The protocol is written once against an ``ops`` object; :class:`DeviceOps`
binds it to the CUDA engine.  The CPU tests bind it to the oracle and run it
over gloo (tests/test_dist_gloo.py).
"""
from __future__ import annotations

import ctypes as C

import torch
import torch.distributed as dist

from . import _lib
from ._lib import check, lib
from .engine import Micro, device_view


def exchange(ops, group=None, comm_device=None) -> int:
    """Run K2..K8 for one rank after ops' compress.  Returns |union|.

    Collectives run on ``ops.device`` tensors (NCCL).  ``comm_device`` (e.g.
    ``"cpu"`` with gloo) stages them through another device instead — used to
    run several ranks' device halves on one GPU in tests."""
    n = dist.get_world_size(group)
    me = dist.get_rank(group)
    dev = ops.device
    cdev = torch.device(comm_device) if comm_device is not None else dev

    def to_c(t):
        return t if t.device == cdev else t.to(cdev)

    def to_d(t):
        return t if t.device == dev else t.to(dev)

    cnt = torch.empty(n, dtype=torch.int64, device=cdev)
    dist.all_gather_into_tensor(cnt, to_c(ops.own_count()), group=group)      # K2
    counts = [int(v) for v in cnt.cpu().tolist()]
    kmax = max(counts)
    if kmax > ops.capacity:  # every rank sees the same counts, so every rank raises
        raise _lib.CapacityError(_lib.MICRO_ECAPACITY,
                                 f"selection of {kmax} exceeds capacity {ops.capacity} on some rank")
    if kmax == 0:
        ops.finalize(None, None, counts, 0)
        return 0
    all_idx = torch.empty(n * kmax, dtype=torch.int32, device=cdev)
    dist.all_gather_into_tensor(all_idx, to_c(ops.own_indices(kmax)), group=group)  # K3
    all_idx = to_d(all_idx)
    send = to_c(ops.gather_foreign(all_idx, counts, kmax))                     # K4
    recv = torch.empty((n - 1) * counts[me], dtype=ops.dtype, device=cdev)
    dist.all_to_all_single(recv, send,                                          # K5
                           output_split_sizes=[0 if r == me else counts[me] for r in range(n)],
                           input_split_sizes=[0 if o == me else counts[o] for o in range(n)],
                           group=group)
    own_sums = to_c(ops.owner_reduce(to_d(recv), counts, kmax))                # K6
    all_sums = torch.empty(n * kmax, dtype=ops.dtype, device=cdev)
    dist.all_gather_into_tensor(all_sums, own_sums, group=group)               # K7
    ops.finalize(all_idx, to_d(all_sums), counts, kmax)                         # K8
    return sum(counts)


class DeviceOps:
    """Binds :func:`exchange` to one rank's `micro_ctx` (n_local == 1)."""

    def __init__(self, m: Micro):
        self.m = m
        self.device, self.dtype = m.device, m.dtype
        self.capacity = m.selection_capacity

    def own_count(self) -> torch.Tensor:
        _, _, cnt = self.m.selection_device(0)
        return cnt

    def own_indices(self, kmax: int) -> torch.Tensor:
        pi, _, _ = self.m.selection_device(0)
        return device_view(pi, kmax, torch.int32, self.device)  # kmax <= selection capacity

    def gather_foreign(self, all_idx, counts, kmax):
        me = self.m.rank
        send = torch.empty(max(sum(counts) - counts[me], 1), dtype=self.dtype, device=self.device)
        hc = (C.c_int64 * len(counts))(*counts)
        check(lib().micro_dist_gather_foreign(self.m.handle, C.c_void_p(all_idx.data_ptr()), hc, kmax,
                                              C.c_void_p(send.data_ptr())))
        return send[: sum(counts) - counts[me]]

    def owner_reduce(self, recv, counts, kmax):
        out = torch.zeros(kmax, dtype=self.dtype, device=self.device)
        hc = (C.c_int64 * len(counts))(*counts)
        check(lib().micro_dist_owner_reduce(self.m.handle, C.c_void_p(recv.data_ptr() if recv.numel() else 0), hc,
                                            C.c_void_p(out.data_ptr())))
        return out

    def finalize(self, all_idx, all_sums, counts, kmax):
        hc = (C.c_int64 * len(counts))(*counts)
        check(lib().micro_dist_finalize(self.m.handle, C.c_void_p(all_idx.data_ptr() if all_idx is not None else 0),
                                        C.c_void_p(all_sums.data_ptr() if all_sums is not None else 0), hc, kmax))


class DistMicro:
    """One rank's MiCRO engine; same calls as :class:`engine.Micro`.

    ``transport="nccl"``: the protocol above (NCCL moves the data).
    ``transport="peer"``: two kernels per rank over peer memory with every
    NVLink transfer contiguous (micro_peer_contribute / _reduce,
    csrc/peer.cuh) between barriers; ``"peer_pull"``: one kernel whose owners
    read the peers' entries remotely (micro_peer_exchange).  The barriers are
    a 4-byte NCCL all-reduce on the compute stream, or, with
    ``comm_device="cpu"`` (tests, several ranks on one GPU), a host barrier
    after a stream sync, so no kernel ever waits on another rank's kernel."""

    def __init__(self, n_g: int, group=None, comm_device=None, transport: str = "nccl", **kw):
        if not dist.is_initialized():
            raise _lib.LogicError(_lib.MICRO_ELOGIC, "torch.distributed is not initialized")
        if transport not in ("nccl", "peer", "peer_pull"):
            raise _lib.InvalidArgument(_lib.MICRO_EINVAL, f"unknown transport {transport!r}")
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.m = Micro(n_g, self.world, n_local=1, rank=self.rank, **kw)
        self.ops = DeviceOps(self.m)
        self.n_g = n_g
        self.comm_device = comm_device
        self.transport = transport
        if transport in ("peer", "peer_pull"):
            self._bar = torch.zeros(1, dtype=torch.int32, device=self.m.device)
            ok, why = True, ""
            try:
                blob = C.create_string_buffer(_lib.MICRO_PEER_HANDLE_BYTES)
                check(lib().micro_peer_export(self.m.handle, blob))
                blobs = [None] * self.world
                dist.all_gather_object(blobs, blob.raw, group=group)
                allb = C.create_string_buffer(b"".join(blobs), _lib.MICRO_PEER_HANDLE_BYTES * self.world)
                check(lib().micro_peer_import(self.m.handle, allb))
            except _lib.MicroError as ex:  # e.g. no peer access between these devices
                ok, why = False, str(ex)
            # every rank must agree on the transport, or the barriers deadlock
            flags = [None] * self.world
            dist.all_gather_object(flags, ok, group=group)
            if not all(flags):
                import warnings
                warnings.warn(f"peer-memory exchange unavailable on some rank ({why or 'remote failure'}); "
                              "falling back to the NCCL protocol")
                self.transport = "nccl"

    def _barrier(self):
        if self.comm_device is not None:  # host barrier (gloo): the stream's work is done first
            self.m.stream.synchronize()
            dist.barrier(group=self.group)
        else:  # stream-ordered: NCCL's stream waits for ours, ours for NCCL's
            with torch.cuda.stream(self.m.stream):
                dist.all_reduce(self._bar, group=self.group)

    def compress(self, grads, eta: float, t: int):
        self.m.compress(grads, eta, t)

    def exchange_timing(self, enable: bool = True):
        """Record CUDA events around the exchange's data movement each step
        (peer: the exchange kernels, barriers excluded; nccl: the whole
        protocol) — the NVLink roofline's denominator in bench.py."""
        self._xt = [] if enable else None

    def exchange_times(self) -> list[float]:
        out = []
        for parts in getattr(self, "_xt", None) or []:
            out.append(sum(a.elapsed_time(b) for a, b in parts))
        return out

    def _timed(self, parts, fn):
        if getattr(self, "_xt", None) is None:
            return fn()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(self.m.stream)
        r = fn()
        b.record(self.m.stream)
        parts.append((a, b))
        return r

    def aggregate(self) -> int | None:
        """NCCL transport: returns |union| (known on the host).  Peer
        transport: asynchronous, returns None (``query().K`` has it)."""
        parts = []
        if getattr(self, "_xt", None) is not None:
            self._xt.append(parts)
        h = self.m.handle
        if self.transport == "peer":  # bulk: every NVLink transfer contiguous
            self._barrier()
            self._timed(parts, lambda: check(lib().micro_peer_contribute(h)))
            self._barrier()
            self._timed(parts, lambda: check(lib().micro_peer_reduce(h)))
            self._barrier()
            check(lib().micro_peer_finalize(h))
            return None
        if self.transport == "peer_pull":  # one kernel: owners read the peers' entries remotely
            self._barrier()
            self._timed(parts, lambda: check(lib().micro_peer_exchange(h)))
            self._barrier()
            check(lib().micro_peer_finalize(h))
            return None
        return self._timed(parts, lambda: exchange(self.ops, self.group, self.comm_device))

    def step(self, grads, eta: float, t: int) -> int | None:
        self.compress(grads, eta, t)
        return self.aggregate()

    def records(self, max_steps: int = 4096) -> list[dict]:
        """IterationRecord scalars (metrics.hpp:15-29) of the whole job: each
        rank holds its own ||e_r|| and delta_r, combined here in rank order
        like the reference's worker loops (harness.cpp:149, :230-235).
        Collective: every rank must call it."""
        recs = self.m.records(max_steps)
        dev = torch.device(self.comm_device) if self.comm_device else self.m.device
        mine = torch.tensor([[r["error_norm"], r["threshold"]] for r in recs] or [[0.0, 0.0]],
                            dtype=torch.float64, device=dev)
        parts = [torch.empty_like(mine) for _ in range(self.world)]
        dist.all_gather(parts, mine, group=self.group)
        cols = [p.cpu().numpy() for p in parts]
        for s, r in enumerate(recs):
            en = th = 0.0
            for c in cols:  # rank order
                en += float(c[s, 0])
                th += float(c[s, 1])
            r["error_norm"], r["threshold"] = en / self.world, th / self.world
        return recs

    def __getattr__(self, name):  # query, history, union, residual, dense, set_model, sync ...
        return getattr(self.m, name)


class GroupMicro:
    """One process driving all n ranks (micro_group_*): rank r's context on
    ``devices[r]`` with its own stream; the exchange runs over direct peer
    pointers with event barriers, so one host thread enqueues the whole
    n-GPU step without blocking."""

    def __init__(self, n_g: int, n: int, devices=None, **kw):
        devices = list(devices) if devices is not None else list(range(n))
        if len(devices) != n:
            raise _lib.InvalidArgument(_lib.MICRO_EINVAL, "one device per rank")
        self.n, self.n_g = n, n_g
        self.streams = [torch.cuda.Stream(device=d) for d in devices]
        self.ranks = [Micro(n_g, n, n_local=1, rank=r, device=devices[r], stream=self.streams[r], **kw)
                      for r in range(n)]
        self._arr = (C.c_void_p * n)(*[m.handle.value for m in self.ranks])
        check(lib().micro_group_attach(self._arr, n))

    def step(self, grads, eta: float, t: int) -> None:
        if len(grads) != self.n:
            raise _lib.InvalidArgument(_lib.MICRO_EINVAL, f"expected {self.n} gradients")
        for m, g in zip(self.ranks, grads):
            m._grads([g])
        self._keep = grads
        ptrs = (C.c_void_p * self.n)(*[g.data_ptr() for g in grads])
        check(lib().micro_group_step(self._arr, self.n, ptrs, eta, t))

    def synchronize(self):
        for s in self.streams:
            s.synchronize()

    def close(self):
        for m in self.ranks:
            m.close()
