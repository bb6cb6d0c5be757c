"""B200-native MiCRO sparsify + aggregate path (arXiv 2310.00967).

The CUDA library (lib/libmicro_b200.so, C ABI in include/micro.h) is the
product; this package is its Python face:

* :mod:`.engine`  — :class:`Micro`, the stateful per-iteration engine
  (run_iteration's MiCRO branch, harness.cpp:121-224).
* :mod:`.sparsim` — the reference's value-level API (partition,
  select_by_threshold, micro_update_threshold, all_gather_indices,
  all_reduce_sparse, accumulate, compensate) on CUDA tensors.
* :mod:`.dist`    — one process per GPU over torch.distributed (NCCL).
"""
from ._lib import (CapacityError, InvalidArgument, LogicError, MicroError,  # noqa: F401
                   NonFiniteGradient, lib)

__all__ = ["Micro", "synth_gaussian", "lib", "MicroError", "InvalidArgument", "LogicError",
           "NonFiniteGradient", "CapacityError"]


def __getattr__(name):
    if name in ("Micro", "synth_gaussian"):
        from . import engine
        return getattr(engine, name)
    raise AttributeError(name)
