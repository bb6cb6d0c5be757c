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


def exchange(ops, group=None, comm_device=None) -> None:
    """Run K2..K8 for one rank after ops' compress (include/micro.h, the
    collective protocol): every buffer has the fixed stride ``ops.kcap`` and
    every count stays on the device, so nothing here waits for the GPU — the
    same protocol nccl_api.cu runs behind the C ABI with NCCL calls.

    Collectives run on ``ops.device`` tensors (NCCL).  ``comm_device`` (e.g.
    ``"cpu"`` with gloo) stages them through another device instead — used to
    run several ranks' device halves on one GPU in tests."""
    dev = ops.device
    cdev = torch.device(comm_device) if comm_device is not None else dev
    b = ops.buffers()

    def all_gather(dst, src):
        if cdev == dev:
            dist.all_gather_into_tensor(dst, src, group=group)
        else:
            out = torch.empty(dst.numel(), dtype=dst.dtype, device=cdev)
            dist.all_gather_into_tensor(out, src.to(cdev), group=group)
            dst.copy_(out)

    def all_to_all(dst, src):  # equal splits: kcap values per pair
        if cdev == dev:
            dist.all_to_all_single(dst, src, group=group)
        else:
            out = torch.empty(dst.numel(), dtype=dst.dtype, device=cdev)
            dist.all_to_all_single(out, src.to(cdev), group=group)
            dst.copy_(out)

    all_gather(b["all_counts"], b["own_count"])   # K2
    all_gather(b["all_idx"], b["own_idx"])        # K3
    ops.gather_foreign()                           # K4
    all_to_all(b["recv"], b["send"])              # K5
    ops.owner_reduce()                             # K6
    all_gather(b["all_sums"], b["own_sums"])      # K7
    ops.finalize()                                 # K8


class DeviceOps:
    """Binds :func:`exchange` to one rank's `micro_ctx` (n_local == 1): the
    library's exchange buffers as torch views, and its device halves."""

    def __init__(self, m: Micro):
        self.m = m
        self.device, self.dtype = m.device, m.dtype
        bd = _lib.micro_dist_bufs()
        check(lib().micro_dist_buffers(m.handle, C.byref(bd)))
        self.kcap = kc = int(bd.kcap)
        n, dev, dt = m.n, m.device, m.dtype
        self._b = {"own_count": device_view(bd.own_count, 1, torch.int64, dev),
                   "own_idx": device_view(bd.own_idx, kc, torch.int32, dev),
                   "all_counts": device_view(bd.all_counts, n, torch.int64, dev),
                   "all_idx": device_view(bd.all_idx, n * kc, torch.int32, dev),
                   "send": device_view(bd.send, n * kc, dt, dev),
                   "recv": device_view(bd.recv, n * kc, dt, dev),
                   "own_sums": device_view(bd.own_sums, kc, dt, dev),
                   "all_sums": device_view(bd.all_sums, n * kc, dt, dev)}

    def buffers(self) -> dict:
        return self._b

    def gather_foreign(self):
        check(lib().micro_dist_gather_foreign(self.m.handle))

    def owner_reduce(self):
        check(lib().micro_dist_owner_reduce(self.m.handle))

    def finalize(self):
        check(lib().micro_dist_finalize(self.m.handle))


class DistMicro:
    """One rank's MiCRO engine; same calls as :class:`engine.Micro`.

    ``transport="nccl"``: the protocol above (NCCL moves the data, through
    torch.distributed).  ``"abi_peer"`` / ``"abi_nccl"``: the same exchanges
    run entirely inside the library over its own NCCL communicator
    (micro_dist_init_nccl + micro_aggregate — what a C++ host calls).
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
        if transport not in ("nccl", "peer", "peer_pull", "abi_peer", "abi_nccl"):
            raise _lib.InvalidArgument(_lib.MICRO_EINVAL, f"unknown transport {transport!r}")
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.m = Micro(n_g, self.world, n_local=1, rank=self.rank, **kw)
        self.ops = DeviceOps(self.m) if transport == "nccl" else None
        self.n_g = n_g
        self.comm_device = comm_device
        self.transport = transport
        if transport in ("abi_peer", "abi_nccl"):
            # the library's own NCCL communicator (micro_dist_init_nccl): rank 0's
            # unique id travels over this process group once
            uid = C.create_string_buffer(_lib.MICRO_NCCL_UNIQUE_ID_BYTES)
            if self.rank == 0:
                check(lib().micro_nccl_unique_id(uid))
            obj = [uid.raw]
            dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group else 0, group=group)
            uid = C.create_string_buffer(obj[0], _lib.MICRO_NCCL_UNIQUE_ID_BYTES)
            check(lib().micro_dist_init_nccl(self.m.handle, uid,
                                             _lib.MICRO_XCHG_PEER if transport == "abi_peer" else _lib.MICRO_XCHG_NCCL))
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
                self.ops = DeviceOps(self.m)

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

    def aggregate(self) -> None:
        """Asynchronous for every transport (``query().K`` has |union|)."""
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
        if self.transport in ("abi_peer", "abi_nccl"):  # the C ABI runs it (nccl_api.cu)
            self._timed(parts, lambda: check(lib().micro_aggregate(h)))
            return None
        with torch.cuda.stream(self.m.stream):  # the collectives ordered with the library's kernels
            self._timed(parts, lambda: exchange(self.ops, self.group, self.comm_device))
        return None

    def step(self, grads, eta: float, t: int) -> None:
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
