"""Host-side face of the MiCRO engine (include/micro.h) for Python callers.

`Micro` owns one `micro_ctx`: either a whole n-worker cluster on one device
(the reference's in-process `ClusterState`, harness.hpp:59-70) or one rank of
an n-GPU job (see dist.py).  All array work runs in the CUDA library; torch is
used only for device memory, streams and tensor views.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Sequence

import numpy as np
import torch

from . import _lib
from ._lib import check, lib

_DT = {torch.float32: _lib.MICRO_F32, torch.float64: _lib.MICRO_F64}
_NP = {torch.float32: np.float32, torch.float64: np.float64}
_TYPESTR = {torch.float32: "<f4", torch.float64: "<f8", torch.int32: "<i4", torch.int64: "<i8"}


class _CudaArray:
    """__cuda_array_interface__ shim: a zero-copy torch view of library memory."""

    def __init__(self, ptr: int, n: int, dtype: torch.dtype):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": _TYPESTR[dtype],
                                         "data": (ptr, False), "version": 3, "strides": None}


def device_view(ptr: int, n: int, dtype: torch.dtype, device: torch.device) -> torch.Tensor:
    if n == 0:
        return torch.empty(0, dtype=dtype, device=device)
    return torch.as_tensor(_CudaArray(ptr, n, dtype), device=device)


def _ptrs(ts: Sequence[torch.Tensor]):
    arr = (C.c_void_p * len(ts))()
    for i, t in enumerate(ts):
        arr[i] = t.data_ptr()
    return arr


@dataclass
class Stats:
    t: int
    steps: int
    K: int
    total_selected: int
    nonfinite: bool
    overflow: bool
    counts: np.ndarray
    deltas: np.ndarray


class Micro:
    """MiCRO sparsify + aggregate for `n_local` workers on one device.

    Parameters mirror SparsifierConfig (sparsifier.hpp:39-46) and
    RunConfig.error_feedback (harness.hpp:46).
    """

    def __init__(self, n_g: int, n_workers: int = 1, *, n_local: int | None = None, rank: int = 0,
                 dtype: torch.dtype = torch.float32, density: float = 0.01,
                 initial_threshold: float = 0.01, scaling_factor: float = 0.01,
                 min_threshold: float = 1e-12, target: str = "split", error_feedback: bool = True,
                 dense_output: bool = True, device: int | torch.device | None = None,
                 stream: torch.cuda.Stream | None = None, selection_capacity: int = 0,
                 record_error_norm: bool = True, sparsifier: str = "micro",
                 grad_dtype: torch.dtype | None = None):
        L = lib()
        if dtype not in _DT:
            raise _lib.InvalidArgument(_lib.MICRO_EINVAL, f"unsupported dtype {dtype}")
        if target not in ("split", "full"):
            raise _lib.InvalidArgument(_lib.MICRO_EINVAL,
                                       f"unknown per-worker target '{target}' (expected split|full)")
        dev = torch.device("cuda", torch.cuda.current_device() if device is None else
                           (device.index if isinstance(device, torch.device) else device))
        cfg = _lib.micro_config()
        L.micro_config_default(C.byref(cfg))
        cfg.n_g, cfg.n_workers = n_g, n_workers
        cfg.n_local = n_workers if n_local is None else n_local
        cfg.rank, cfg.dtype = rank, _DT[dtype]
        cfg.density, cfg.initial_threshold = density, initial_threshold
        cfg.scaling_factor, cfg.min_threshold = scaling_factor, min_threshold
        cfg.target = 0 if target == "split" else 1
        cfg.error_feedback, cfg.dense_output = int(error_feedback), int(dense_output)
        cfg.device, cfg.selection_capacity = dev.index, selection_capacity
        cfg.record_error_norm = int(record_error_norm)
        if sparsifier not in _lib.SPARSIFIERS:
            raise _lib.InvalidArgument(_lib.MICRO_EINVAL, f"unknown sparsifier '{sparsifier}'")
        cfg.sparsifier = _lib.SPARSIFIERS[sparsifier]
        # grad_dtype=torch.float32 with dtype=torch.float64: fp32 gradients into
        # fp64 state and arithmetic (include/micro.h micro_config.grad_dtype)
        grad_dtype = dtype if grad_dtype is None else grad_dtype
        if grad_dtype != dtype and not (grad_dtype == torch.float32 and dtype == torch.float64):
            raise _lib.InvalidArgument(_lib.MICRO_EINVAL, f"gradients of {grad_dtype} need state of the same dtype "
                                                          f"(or float32 gradients into float64 state), not {dtype}")
        cfg.grad_dtype = 0 if grad_dtype == dtype else _lib.MICRO_GRAD_F32
        self.grad_dtype = grad_dtype
        self.sparsifier = sparsifier
        self.cfg = cfg
        self.device, self.dtype = dev, dtype
        self.n_g, self.n, self.n_local, self.rank = n_g, n_workers, cfg.n_local, rank
        max_range = n_g if sparsifier != "micro" else -(-n_g // max(n_workers, 1))
        self.selection_capacity = min(selection_capacity, max_range) if selection_capacity else max_range
        with torch.cuda.device(dev):
            self.stream = stream or torch.cuda.current_stream(dev)
        h = C.c_void_p()
        check(L.micro_ctx_create(C.byref(h), C.byref(cfg), C.c_void_p(self.stream.cuda_stream)))
        self._h = h
        self._model = None

    # -- lifecycle ---------------------------------------------------------
    def close(self):
        if getattr(self, "_h", None):
            lib().micro_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def reset(self):
        check(lib().micro_ctx_reset(self._h))

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def set_model(self, x: torch.Tensor | None):
        if x is not None:
            assert x.is_cuda and x.dtype == self.dtype and x.numel() == self.n_g and x.is_contiguous()
        self._model = x
        check(lib().micro_set_model(self._h, C.c_void_p(x.data_ptr() if x is not None else 0)))

    # -- the step ------------------------------------------------------------
    def _grads(self, grads):
        if isinstance(grads, torch.Tensor):
            grads = [grads] if grads.dim() == 1 else list(grads)
        if len(grads) != self.n_local:
            raise _lib.InvalidArgument(_lib.MICRO_EINVAL, f"expected {self.n_local} gradients, got {len(grads)}")
        for g in grads:
            if not (g.is_cuda and g.dtype == self.grad_dtype and g.numel() == self.n_g and g.is_contiguous()):
                raise _lib.InvalidArgument(_lib.MICRO_EINVAL,
                                           f"gradient must be a contiguous {self.grad_dtype} CUDA tensor of {self.n_g}")
        return grads

    def compress(self, grads, eta: float, t: int):
        grads = self._grads(grads)
        self._keep = grads
        check(lib().micro_compress(self._h, _ptrs(grads), eta, t))

    def aggregate(self):
        check(lib().micro_aggregate(self._h))

    def step(self, grads, eta: float, t: int):
        grads = self._grads(grads)
        self._keep = grads
        check(lib().micro_step(self._h, _ptrs(grads), eta, t))

    def step_host(self, h_grads: torch.Tensor, eta: float, t: int, out_idx: np.ndarray | None = None,
                  out_sums: np.ndarray | None = None):
        """End-to-end call with host buffers (pinned CPU tensor of n_local*n_g)."""
        assert not h_grads.is_cuda and h_grads.dtype == self.grad_dtype and h_grads.is_contiguous()
        own = out_idx is None or out_sums is None
        if own:
            out_idx, out_sums = self._host_out()
        K = C.c_int64()
        check(lib().micro_step_host(self._h, C.c_void_p(h_grads.data_ptr()), eta, t,
                                    out_idx.ctypes.data, out_sums.ctypes.data, min(out_idx.size, out_sums.size),
                                    C.byref(K)))
        if own:  # the internal buffers are reused by the next call
            return out_idx[: K.value].copy(), out_sums[: K.value].copy()
        return out_idx[: K.value], out_sums[: K.value]

    def _host_out(self):
        """Pinned result buffers (n_g entries), allocated once per context:
        full-bandwidth D2H; results are copied out of them (K entries)."""
        if getattr(self, "_hout", None) is None:
            pin = torch.cuda.is_available()
            ti = torch.empty(self.n_g, dtype=torch.int32, pin_memory=pin)
            ts = torch.empty(self.n_g, dtype=self.dtype, pin_memory=pin)
            self._hout = (ti, ts)
        ti, ts = self._hout
        return ti.numpy(), ts.numpy()

    def sync(self):
        check(lib().micro_sync(self._h))

    # -- results ---------------------------------------------------------------
    def query(self) -> Stats:
        st = _lib.micro_stats()
        counts = np.empty(self.n_local, np.int64)
        deltas = np.empty(self.n_local, np.float64)
        check(lib().micro_query(self._h, C.byref(st), counts.ctypes.data, deltas.ctypes.data))
        return Stats(st.t, st.steps, st.K, st.total_selected, bool(st.nonfinite), bool(st.overflow),
                     counts, deltas)

    def history(self, max_steps: int = 4096) -> dict:
        n = min(max_steps, 4096)
        t = np.empty(n, np.int64)
        K = np.empty(n, np.int64)
        cnt = np.empty(n * self.n_local, np.int64)
        dl = np.empty(n * self.n_local, np.float64)
        w = C.c_int64()
        check(lib().micro_history(self._h, n, t.ctypes.data, K.ctypes.data, cnt.ctypes.data,
                                  dl.ctypes.data, C.byref(w)))
        m = w.value
        return dict(t=t[:m], K=K[:m], counts=cnt[: m * self.n_local].reshape(m, self.n_local),
                    delta_used=dl[: m * self.n_local].reshape(m, self.n_local))

    def records(self, max_steps: int = 4096) -> list[dict]:
        """The reference's IterationRecord scalars (metrics.hpp:15-29) of the
        last steps, oldest first: t, actual_density, buildup_factor,
        redundant_traffic_factor, error_norm, threshold (+ K, total_selected)."""
        n = min(max_steps, 4096)
        buf = (_lib.micro_record * max(n, 1))()
        w = C.c_int64()
        check(lib().micro_records(self._h, n, buf, C.byref(w)))
        return [{f: getattr(buf[i], f) for f, _ in _lib.micro_record._fields_} for i in range(w.value)]

    def kernel_timing(self, enable: bool = True, every: int = 1):
        """Record CUDA-event durations of K1's streaming pass (diagnostics),
        every `every`-th launch."""
        check(lib().micro_kernel_timing(self._h, every if enable else 0))

    def kernel_times(self, max_n: int = 1024) -> np.ndarray:
        out = np.empty(max_n, np.float32)
        w = C.c_int32()
        check(lib().micro_kernel_times(self._h, out.ctypes.data, max_n, C.byref(w)))
        return out[: w.value].copy()

    def union(self, out_idx: np.ndarray | None = None, out_sums: np.ndarray | None = None):
        """(indices int32, sums) of the last step as host numpy arrays; with
        caller buffers (e.g. pinned) the result views them without a copy."""
        if out_idx is None or out_sums is None:
            idx, sums = self._host_out()
        else:
            idx, sums = out_idx, out_sums
        K = C.c_int64()
        check(lib().micro_copy_union(self._h, idx.ctypes.data, sums.ctypes.data, min(idx.size, sums.size),
                                     C.byref(K)))
        if out_idx is None or out_sums is None:
            return idx[: K.value].copy(), sums[: K.value].copy()
        return idx[: K.value], sums[: K.value]

    def union_device(self):
        """Zero-copy device views (valid until the next step): idx, sums, K tensor."""
        pi, ps, pk = C.c_void_p(), C.c_void_p(), C.c_void_p()
        check(lib().micro_union_device(self._h, C.byref(pi), C.byref(ps), C.byref(pk)))
        Kt = device_view(pk.value, 1, torch.int64, self.device)
        return pi.value, ps.value, Kt

    def residual(self, i: int = 0) -> np.ndarray:
        out = np.empty(self.n_g, _NP[self.dtype])
        check(lib().micro_copy_residual(self._h, i, out.ctypes.data))
        return out

    def residual_device(self, i: int = 0) -> torch.Tensor:
        p = C.c_void_p()
        check(lib().micro_residual_device(self._h, i, C.byref(p)))
        return device_view(p.value, self.n_g, self.dtype, self.device)

    def dense(self) -> np.ndarray:
        out = np.empty(self.n_g, _NP[self.dtype])
        check(lib().micro_copy_dense(self._h, out.ctypes.data))
        return out

    def dense_device(self) -> torch.Tensor:
        p = C.c_void_p()
        check(lib().micro_dense_device(self._h, C.byref(p)))
        return device_view(p.value, self.n_g, self.dtype, self.device)

    def selection_device(self, i: int = 0):
        """Own selection of local worker i after compress: (idx ptr, val ptr, count view)."""
        pi, pv, pc = C.c_void_p(), C.c_void_p(), C.c_void_p()
        check(lib().micro_selection_device(self._h, i, C.byref(pi), C.byref(pv), C.byref(pc)))
        return pi.value, pv.value, device_view(pc.value, 1, torch.int64, self.device)

    def thresholds_device(self) -> torch.Tensor:
        p = C.c_void_p()
        check(lib().micro_threshold_device(self._h, C.byref(p)))
        return device_view(p.value, self.n_local, torch.float64, self.device)


def synth_gaussian(out: torch.Tensor, seed: int, worker: int, t: int, stream: torch.cuda.Stream | None = None):
    """Fill `out` (CUDA fp32/fp64) with the include/micro_synth.h gradients."""
    s = stream or torch.cuda.current_stream(out.device)
    check(lib().micro_synth_gaussian(_DT[out.dtype], seed, worker, t, out.numel(), C.c_void_p(out.data_ptr()),
                                     C.c_void_p(s.cuda_stream)))
    return out
