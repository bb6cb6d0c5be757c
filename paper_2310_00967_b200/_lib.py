"""ctypes binding of the in-tree CUDA library (lib/libmicro_b200.so).

The product has no CPU path: if the library is missing this module raises
on first use instead of falling back to anything.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "lib", "libmicro_b200.so")

I32, I64, U32, U64, DBL, VP = C.c_int32, C.c_int64, C.c_uint32, C.c_uint64, C.c_double, C.c_void_p
PI64, PU64, PDBL = C.POINTER(I64), C.POINTER(U64), C.POINTER(DBL)

MICRO_OK, MICRO_EINVAL, MICRO_ELOGIC, MICRO_ENONFINITE = 0, 1, 2, 3
MICRO_ECUDA, MICRO_ENCCL, MICRO_ECAPACITY, MICRO_ENOMEM = 4, 5, 6, 7
MICRO_F32, MICRO_F64 = 0, 1
MICRO_MAX_WORKERS = 64
MICRO_PEER_HANDLE_BYTES = 640
SPARSIFIERS = {"micro": 0, "topk": 1, "cltk": 2, "hard": 3, "dense": 4}  # sparsifier.hpp:21


class micro_config(C.Structure):
    _fields_ = [
        ("n_g", I64), ("n_workers", I32), ("n_local", I32), ("rank", I32), ("dtype", I32),
        ("density", DBL), ("initial_threshold", DBL), ("scaling_factor", DBL), ("min_threshold", DBL),
        ("target", I32), ("error_feedback", I32), ("dense_output", I32), ("device", I32),
        ("selection_capacity", I64), ("record_error_norm", I32), ("sparsifier", I32), ("grad_dtype", I32),
    ]


class micro_stats(C.Structure):
    _fields_ = [("t", I64), ("steps", I64), ("K", I64), ("total_selected", I64),
                ("nonfinite", I32), ("overflow", I32)]


class micro_record(C.Structure):
    _fields_ = [("t", I64), ("K", I64), ("total_selected", I64), ("actual_density", DBL),
                ("buildup_factor", DBL), ("redundant_traffic_factor", DBL), ("error_norm", DBL),
                ("threshold", DBL)]


class micro_dist_bufs(C.Structure):
    _fields_ = [("kcap", I64), ("own_count", VP), ("own_idx", VP), ("all_counts", VP), ("all_idx", VP),
                ("send", VP), ("recv", VP), ("own_sums", VP), ("all_sums", VP)]


MICRO_NCCL_UNIQUE_ID_BYTES = 128
MICRO_XCHG_PEER, MICRO_XCHG_NCCL = 0, 1
MICRO_GRAD_SAME, MICRO_GRAD_F32 = 0, 1  # micro_config.grad_dtype


class MicroError(RuntimeError):
    """Base of the status-code exceptions (include/micro.h)."""

    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class InvalidArgument(MicroError, ValueError):
    """std::invalid_argument (MICRO_EINVAL)."""


class LogicError(MicroError):
    """std::logic_error (MICRO_ELOGIC)."""


class NonFiniteGradient(MicroError):
    """std::runtime_error for a non-finite gradient (MICRO_ENONFINITE)."""


class CudaError(MicroError):
    pass


class CapacityError(MicroError):
    pass


_EXC = {MICRO_EINVAL: InvalidArgument, MICRO_ELOGIC: LogicError, MICRO_ENONFINITE: NonFiniteGradient,
        MICRO_ECUDA: CudaError, MICRO_ENCCL: CudaError, MICRO_ECAPACITY: CapacityError,
        MICRO_ENOMEM: CudaError}

_lib = None
_lock = threading.Lock()

_SIGS = {
    "micro_abi_version": ([], I32),
    "micro_status_string": ([I32], C.c_char_p),
    "micro_last_error": ([], C.c_char_p),
    "micro_partition": ([I64, I32, I64, I32, PI64, PI64], I32),
    "micro_global_target_count": ([DBL, I64, PU64], I32),
    "micro_per_worker_target_count": ([DBL, I64, I32, I32, PU64], I32),
    "micro_update_threshold": ([PDBL, U64, U64, DBL, DBL], I32),
    "micro_accumulate": ([I32, VP, DBL, VP, VP, I64, VP], I32),
    "micro_select_by_threshold": ([I32, VP, I64, I64, I64, DBL, VP, VP, I64, VP, VP], I32),
    "micro_compensate": ([I32, VP, I64, VP, I64, VP], I32),
    "micro_select_topk": ([I32, VP, I64, I64, I64, I64, VP, VP, I64, VP, VP], I32),
    "micro_all_reduce_sparse_values": ([I32, C.POINTER(VP), I32, I64, VP, I64, VP, VP], I32),
    "micro_all_reduce_sparse": ([I32, C.POINTER(VP), I32, I64, VP, I64, VP, VP], I32),
    "micro_all_gather_indices": ([I32, PI64, VP, VP, PI64, VP], I32),
    "micro_error_metric": ([I32, C.POINTER(VP), I32, I64, PDBL, VP], I32),
    "micro_synth_gaussian": ([I32, U64, U32, U64, I64, VP, VP], I32),
    "micro_device_malloc": ([C.POINTER(VP), I64, I32], I32),
    "micro_value_workspace_trim": ([I32], I32),
    "micro_device_free": ([VP], I32),
    "micro_host_malloc": ([C.POINTER(VP), I64], I32),
    "micro_host_free": ([VP], I32),
    "micro_memcpy": ([VP, VP, I64, I32, VP], I32),
    "micro_device_count": ([C.POINTER(I32)], I32),
    "micro_config_default": ([C.POINTER(micro_config)], None),
    "micro_ctx_create": ([C.POINTER(VP), C.POINTER(micro_config), VP], I32),
    "micro_ctx_destroy": ([VP], I32),
    "micro_ctx_reset": ([VP], I32),
    "micro_ctx_stream": ([VP], VP),
    "micro_set_model": ([VP, VP], I32),
    "micro_compress": ([VP, C.POINTER(VP), DBL, I64], I32),
    "micro_aggregate": ([VP], I32),
    "micro_step": ([VP, C.POINTER(VP), DBL, I64], I32),
    "micro_step_host": ([VP, VP, DBL, I64, VP, VP, I64, PI64], I32),
    "micro_sync": ([VP], I32),
    "micro_query": ([VP, C.POINTER(micro_stats), VP, VP], I32),
    "micro_history": ([VP, I64, VP, VP, VP, VP, PI64], I32),
    "micro_records": ([VP, I64, VP, PI64], I32),
    "micro_kernel_timing": ([VP, I32], I32),
    "micro_kernel_times": ([VP, VP, I32, C.POINTER(I32)], I32),
    "micro_union_device": ([VP, C.POINTER(VP), C.POINTER(VP), C.POINTER(VP)], I32),
    "micro_dense_device": ([VP, C.POINTER(VP)], I32),
    "micro_residual_device": ([VP, I32, C.POINTER(VP)], I32),
    "micro_selection_device": ([VP, I32, C.POINTER(VP), C.POINTER(VP), C.POINTER(VP)], I32),
    "micro_threshold_device": ([VP, C.POINTER(VP)], I32),
    "micro_copy_union": ([VP, VP, VP, I64, PI64], I32),
    "micro_copy_residual": ([VP, I32, VP], I32),
    "micro_copy_dense": ([VP, VP], I32),
    "micro_dist_buffers": ([VP, C.POINTER(micro_dist_bufs)], I32),
    "micro_dist_gather_foreign": ([VP], I32),
    "micro_dist_owner_reduce": ([VP], I32),
    "micro_dist_finalize": ([VP], I32),
    "micro_nccl_unique_id": ([VP], I32),
    "micro_set_device": ([I32], I32),
    "micro_dist_init_nccl": ([VP, VP, I32], I32),
    "micro_dist_attach_nccl": ([VP, VP, I32], I32),
    "micro_peer_export": ([VP, VP], I32),
    "micro_peer_import": ([VP, VP], I32),
    "micro_peer_exchange": ([VP], I32),
    "micro_peer_finalize": ([VP], I32),
    "micro_peer_contribute": ([VP], I32),
    "micro_peer_reduce": ([VP], I32),
    "micro_group_attach": ([C.POINTER(VP), I32], I32),
    "micro_group_step": ([C.POINTER(VP), I32, C.POINTER(VP), DBL, I64], I32),
}

EXPORTED = sorted(_SIGS)


def lib() -> C.CDLL:
    """Load the CUDA library (once).  Raises ImportError when it is absent:
    there is deliberately no fallback."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(
                    f"{LIB_PATH} is missing: build it with `python -m paper_2310_00967_b200.build` "
                    "(the MiCRO path has no CPU fallback)")
            L = C.CDLL(LIB_PATH)
            for name, (args, res) in _SIGS.items():
                f = getattr(L, name)
                f.argtypes = args
                f.restype = res
            if L.micro_abi_version() != 5:
                raise ImportError("libmicro_b200.so ABI version mismatch")
            _lib = L
    return _lib


def check(rc: int) -> None:
    if rc != MICRO_OK:
        msg = lib().micro_last_error().decode(errors="replace")
        raise _EXC.get(rc, MicroError)(rc, msg)
