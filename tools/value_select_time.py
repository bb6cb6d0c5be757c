"""Time the value-level select_by_threshold (the reference's
sparsifier.cpp:22-37 call on a device array) at C3 size: through the Python
face (allocates its outputs, reads the count back) and through the C ABI
with preallocated outputs (stream-ordered, no host sync per call)."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_00967_b200 import sparsim as S  # noqa: E402
from paper_2310_00967_b200._lib import MICRO_F32, MICRO_F64, check, lib  # noqa: E402

n, delta, reps = 138_000_000, 0.0258, 50
for dt in (torch.float64, torch.float32, torch.float64):
    acc = torch.randn(n, device="cuda", dtype=dt) * 0.01
    rng = S.PartitionRange(0, n, 0)
    for _ in range(3):
        S.select_by_threshold(acc, rng, delta)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        sel = S.select_by_threshold(acc, rng, delta)
    b.record()
    torch.cuda.synchronize()
    us_py = a.elapsed_time(b) / reps * 1e3
    k = sel.count()
    idx = torch.empty(n, dtype=torch.int32, device="cuda")
    val = torch.empty(n, dtype=dt, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    code = MICRO_F64 if dt == torch.float64 else MICRO_F32

    def call():
        check(lib().micro_select_by_threshold(code, C.c_void_p(acc.data_ptr()), n, 0, n, delta,
                                              C.c_void_p(idx.data_ptr()), C.c_void_p(val.data_ptr()), n,
                                              C.c_void_p(cnt.data_ptr()), C.c_void_p(st)))
    for _ in range(3):
        call()
    torch.cuda.synchronize()
    a.record()
    for _ in range(reps):
        call()
    b.record()
    torch.cuda.synchronize()
    us_c = a.elapsed_time(b) / reps * 1e3
    byts = n * acc.element_size() + k * (4 + acc.element_size())
    print(f"{dt}: select_by_threshold over {n} elements, k = {k}: Python face {us_py:.1f} us/call; C ABI "
          f"(stream-ordered) {us_c:.1f} us/call = {byts / us_c / 1e3:.0f} GB/s algorithmic "
          f"(acc read once + the pairs)")
