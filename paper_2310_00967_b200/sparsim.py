"""The reference's value-level sparsifier API (namespace ``sparsim``) on CUDA
tensors, backed by the C ABI.  Same names, argument meaning and error
behaviour as /root/reference/proj/include/sparsim/*.hpp:

  partition                 tensor.hpp:48-63
  select_by_threshold       sparsifier.hpp:49-50 / sparsifier.cpp:22-37
  micro_update_threshold    sparsifier.hpp:59-61 / sparsifier.cpp:69-83
  global_target_count       sparsifier.cpp:110-116
  per_worker_target_count   sparsifier.cpp:118-125
  accumulate / compensate   error_feedback.hpp:17-39
  all_gather_indices        collectives.cpp:14-28
  all_reduce_sparse(_values) collectives.cpp:30-57
  buildup_factor / redundant_traffic_factor  collectives.cpp:59-69
  actual_density            metrics.cpp:7-10

std::invalid_argument surfaces as :class:`InvalidArgument` (a ValueError),
std::logic_error as :class:`LogicError`, the non-finite runtime_error as
:class:`NonFiniteGradient`.  Indices on the device are int32 (n_g < 2^31).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Sequence

import torch

from . import _lib
from ._lib import InvalidArgument, check, lib

_DT = {torch.float32: _lib.MICRO_F32, torch.float64: _lib.MICRO_F64}


def _stream(dev):
    return C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def _vec(v: torch.Tensor, what: str) -> torch.Tensor:
    if not isinstance(v, torch.Tensor) or not v.is_cuda or v.dtype not in _DT or v.dim() != 1:
        raise InvalidArgument(_lib.MICRO_EINVAL, f"{what}: expected a 1-D float32/float64 CUDA tensor")
    return v.contiguous()


@dataclass(frozen=True)
class PartitionRange:
    """tensor.hpp:25-32"""
    start: int = 0
    end: int = 0
    owner: int = 0

    def size(self) -> int:
        return self.end - self.start


@dataclass
class SparseSelection:
    """sparsifier.hpp:28-33 — strictly increasing global indices + acc values."""
    indices: torch.Tensor
    values: torch.Tensor

    def count(self) -> int:
        return int(self.indices.numel())


@dataclass
class ThresholdState:
    """sparsifier.hpp:35-37"""
    delta: float = 0.0


@dataclass
class SparsifierConfig:
    """sparsifier.hpp:39-46 (MiCRO fields)."""
    kind: str = "micro"
    density: float = 0.01
    initial_threshold: float = 0.01
    scaling_factor: float = 0.01
    min_threshold: float = 1e-12
    target: str = "split"


@dataclass
class AggregatedSelection:
    """collectives.hpp:15-20"""
    indices: torch.Tensor
    per_worker_counts: list = field(default_factory=list)

    def total_selected(self) -> int:
        return int(sum(self.per_worker_counts))


def partition(n_g: int, n: int, t: int, worker: int) -> PartitionRange:
    s, e = C.c_int64(), C.c_int64()
    check(lib().micro_partition(n_g, n, t, worker, C.byref(s), C.byref(e)))
    return PartitionRange(s.value, e.value, worker)


def global_target_count(density: float, n_g: int) -> int:
    k = C.c_uint64()
    check(lib().micro_global_target_count(density, n_g, C.byref(k)))
    return k.value


def per_worker_target_count(density: float, n_g: int, n: int, target: str = "split") -> int:
    if target not in ("split", "full"):
        raise InvalidArgument(_lib.MICRO_EINVAL, f"unknown per-worker target '{target}' (expected split|full)")
    k = C.c_uint64()
    check(lib().micro_per_worker_target_count(density, n_g, n, 0 if target == "split" else 1, C.byref(k)))
    return k.value


def micro_update_threshold(state: ThresholdState, k_target: int, k_selected: int, alpha: float,
                           min_threshold: float = 1e-12) -> ThresholdState:
    d = C.c_double(state.delta)
    check(lib().micro_update_threshold(C.byref(d), k_target, k_selected, alpha, min_threshold))
    return ThresholdState(d.value)


def accumulate(residual: torch.Tensor, eta: float, grad: torch.Tensor) -> torch.Tensor:
    residual, grad = _vec(residual, "accumulate"), _vec(grad, "accumulate")
    if residual.numel() != grad.numel():
        raise InvalidArgument(_lib.MICRO_EINVAL,
                              f"accumulate: length mismatch ({residual.numel()} vs {grad.numel()})")
    if residual.dtype != grad.dtype:
        raise InvalidArgument(_lib.MICRO_EINVAL, "accumulate: dtype mismatch")
    out = torch.empty_like(residual)
    check(lib().micro_accumulate(_DT[residual.dtype], C.c_void_p(residual.data_ptr()), eta,
                                 C.c_void_p(grad.data_ptr()), C.c_void_p(out.data_ptr()), residual.numel(),
                                 _stream(residual.device)))
    return out


def select_by_threshold(acc: torch.Tensor, rng: PartitionRange, delta: float) -> SparseSelection:
    acc = _vec(acc, "selection")
    if acc.data_ptr() % 16:
        acc = acc.clone()
    m = max(rng.end - rng.start, 0)
    idx = torch.empty(max(m, 1), dtype=torch.int32, device=acc.device)
    val = torch.empty(max(m, 1), dtype=acc.dtype, device=acc.device)
    cnt = torch.zeros(1, dtype=torch.int64, device=acc.device)
    check(lib().micro_select_by_threshold(_DT[acc.dtype], C.c_void_p(acc.data_ptr()), acc.numel(), rng.start,
                                          rng.end, delta, C.c_void_p(idx.data_ptr()), C.c_void_p(val.data_ptr()),
                                          m, C.c_void_p(cnt.data_ptr()), _stream(acc.device)))
    k = int(cnt.item())
    return SparseSelection(idx[:k], val[:k])


def select_topk(acc: torch.Tensor, rng: PartitionRange, k: int) -> SparseSelection:
    """sparsifier.cpp:39-67: the k largest |acc| in the range, ties to the lower index, ascending."""
    acc = _vec(acc, "select_topk")
    if acc.data_ptr() % 16:
        acc = acc.clone()
    m = max(rng.end - rng.start, 0)
    idx = torch.empty(max(k, 1), dtype=torch.int32, device=acc.device)
    val = torch.empty(max(k, 1), dtype=acc.dtype, device=acc.device)
    cnt = torch.zeros(1, dtype=torch.int64, device=acc.device)
    check(lib().micro_select_topk(_DT[acc.dtype], C.c_void_p(acc.data_ptr()), acc.numel(), rng.start, rng.end, k,
                                  C.c_void_p(idx.data_ptr()), C.c_void_p(val.data_ptr()), max(k, 0),
                                  C.c_void_p(cnt.data_ptr()), _stream(acc.device)))
    n = int(cnt.item())
    return SparseSelection(idx[:n], val[:n])


def cltk_select(acc_leader: torch.Tensor, k_total: int, leader: int, t: int, n: int) -> SparseSelection:
    """sparsifier.cpp:85-97: the cycling leader's global top-k."""
    if n < 1 or leader < 0 or leader >= n:
        raise InvalidArgument(_lib.MICRO_EINVAL, "cltk_select: leader id out of range")
    if t < 0 or t % n != leader:
        raise _lib.LogicError(_lib.MICRO_ELOGIC, f"cltk_select: worker {leader} is not the leader at iteration {t} "
                                                 "(leader cycles as t mod n)")
    acc_leader = _vec(acc_leader, "cltk_select")
    if k_total > acc_leader.numel():
        raise InvalidArgument(_lib.MICRO_EINVAL, "cltk_select: k exceeds gradient count")
    return select_topk(acc_leader, PartitionRange(0, acc_leader.numel(), leader), k_total)


def select_all(acc: torch.Tensor) -> SparseSelection:
    """sparsifier.cpp:103-108: every index, including zeros."""
    acc = _vec(acc, "select_all")
    return SparseSelection(torch.arange(acc.numel(), dtype=torch.int32, device=acc.device), acc.clone())


def hard_threshold_select(acc: torch.Tensor, delta_fixed: float) -> SparseSelection:
    """sparsifier.cpp:98-100 — the fixed-threshold baseline over the whole vector."""
    return select_by_threshold(acc, PartitionRange(0, acc.numel(), 0), delta_fixed)


def compensate(acc: torch.Tensor, selected) -> torch.Tensor:
    acc = _vec(acc, "compensate")
    idx = selected.indices if isinstance(selected, SparseSelection) else torch.as_tensor(selected)
    idx = idx.to(device=acc.device, dtype=torch.int32).contiguous()
    out = acc.clone()
    check(lib().micro_compensate(_DT[acc.dtype], C.c_void_p(out.data_ptr()), out.numel(),
                                 C.c_void_p(idx.data_ptr()), idx.numel(), _stream(acc.device)))
    return out


def all_gather_indices(selections: Sequence[SparseSelection]) -> AggregatedSelection:
    counts = [s.count() for s in selections]
    dev = selections[0].indices.device if selections else torch.device("cuda")
    total = sum(counts)
    cat = (torch.cat([s.indices.to(torch.int32) for s in selections]) if total
           else torch.empty(1, dtype=torch.int32, device=dev)).contiguous()
    out = torch.empty(max(total, 1), dtype=torch.int32, device=dev)
    hc = (C.c_int64 * max(len(counts), 1))(*counts)
    K = C.c_int64()
    check(lib().micro_all_gather_indices(len(counts), hc, C.c_void_p(cat.data_ptr()), C.c_void_p(out.data_ptr()),
                                         C.byref(K), _stream(dev)))
    return AggregatedSelection(out[: K.value], counts)


def _accs(accumulators):
    if len(accumulators) == 0:
        raise InvalidArgument(_lib.MICRO_EINVAL, "all_reduce_sparse: no workers")
    accs = [_vec(a, "all_reduce_sparse") for a in accumulators]
    n_g = accs[0].numel()
    if any(a.numel() != n_g for a in accs):
        raise InvalidArgument(_lib.MICRO_EINVAL, "all_reduce_sparse: accumulator length mismatch")
    if any(a.dtype != accs[0].dtype for a in accs):
        raise InvalidArgument(_lib.MICRO_EINVAL, "all_reduce_sparse: dtype mismatch")
    arr = (C.c_void_p * len(accs))(*[a.data_ptr() for a in accs])
    return accs, arr, n_g


def all_reduce_sparse_values(accumulators, agg: AggregatedSelection) -> torch.Tensor:
    accs, arr, n_g = _accs(accumulators)
    u = agg.indices.to(device=accs[0].device, dtype=torch.int32).contiguous()
    out = torch.empty(max(u.numel(), 1), dtype=accs[0].dtype, device=accs[0].device)
    check(lib().micro_all_reduce_sparse_values(_DT[accs[0].dtype], arr, len(accs), n_g, C.c_void_p(u.data_ptr()),
                                               u.numel(), C.c_void_p(out.data_ptr()), _stream(u.device)))
    return out[: u.numel()]


def all_reduce_sparse(accumulators, agg: AggregatedSelection) -> torch.Tensor:
    accs, arr, n_g = _accs(accumulators)
    u = agg.indices.to(device=accs[0].device, dtype=torch.int32).contiguous()
    out = torch.empty(n_g, dtype=accs[0].dtype, device=accs[0].device)
    check(lib().micro_all_reduce_sparse(_DT[accs[0].dtype], arr, len(accs), n_g, C.c_void_p(u.data_ptr()),
                                        u.numel(), C.c_void_p(out.data_ptr()), _stream(u.device)))
    return out


def buildup_factor(agg: AggregatedSelection, k_target_global: int) -> float:
    if agg.total_selected() == 0:
        return 0.0
    if k_target_global == 0:
        raise InvalidArgument(_lib.MICRO_EINVAL, "buildup_factor: zero target count")
    return agg.indices.numel() / k_target_global


def redundant_traffic_factor(agg: AggregatedSelection) -> float:
    tot = agg.total_selected()
    return 0.0 if tot == 0 else tot / agg.indices.numel()


def actual_density(agg: AggregatedSelection, n_g: int) -> float:
    if n_g < 1:
        raise InvalidArgument(_lib.MICRO_EINVAL, "actual_density: n_g must be positive")
    return agg.indices.numel() / n_g


def error_metric(residuals) -> float:
    """error_feedback.hpp:41-48: (sum_i ||e_i||_2) / n, norms summed in worker
    order (each ||e_i||^2 a deterministic fp64 tree sum on the device)."""
    if len(residuals) == 0:
        raise InvalidArgument(_lib.MICRO_EINVAL, "error_metric: no workers")
    res = [_vec(r, "error_metric") for r in residuals]
    if any(r.numel() != res[0].numel() or r.dtype != res[0].dtype for r in res):
        raise InvalidArgument(_lib.MICRO_EINVAL, "error_metric: residuals must share length and dtype")
    arr = (C.c_void_p * len(res))(*[r.data_ptr() for r in res])
    out = C.c_double()
    check(lib().micro_error_metric(_DT[res[0].dtype], arr, len(res), res[0].numel(), C.byref(out),
                                   _stream(res[0].device)))
    return out.value


@dataclass(frozen=True)
class LrSchedule:
    """harness.hpp:25-32: step decay of the learning rate eta(t)."""
    initial: float = 0.01
    decay_factor: float = 0.1
    decay_at: int = -1  # -1: 3/4 of the run


def resolve_decay_at(lr: LrSchedule, iterations: int) -> int:
    """harness.cpp:109-110."""
    return lr.decay_at if lr.decay_at >= 0 else (3 * iterations) // 4


def learning_rate_at(lr: LrSchedule, decay_at: int, t: int) -> float:
    """harness.cpp:61-63: the eta handed to each MiCRO step (host arithmetic)."""
    return lr.initial * (lr.decay_factor if t >= decay_at else 1.0)


# sparsifier.cpp:127-160: the kind / target names of the reference's CLI and records
SPARSIFIER_KINDS = ("micro", "topk", "cltk", "hard", "dense")


def parse_sparsifier_kind(name: str) -> str:
    if name == "hard_threshold":
        return "hard"
    if name not in SPARSIFIER_KINDS:
        raise InvalidArgument(_lib.MICRO_EINVAL, f"unknown sparsifier '{name}' (expected micro|topk|cltk|hard|dense)")
    return name


def parse_per_worker_target(name: str) -> str:
    if name not in ("split", "full"):
        raise InvalidArgument(_lib.MICRO_EINVAL, f"unknown per-worker target '{name}' (expected split|full)")
    return name
