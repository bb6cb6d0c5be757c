"""Time the value-level select_by_threshold (sparsim.select_by_threshold on a
device tensor: the reference's sparsifier.cpp:22-37 call) at C3 size."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_00967_b200 import sparsim as S  # noqa: E402

for dt in (torch.float32, torch.float64):
    n = 138_000_000
    acc = torch.randn(n, device="cuda", dtype=dt) * 0.01
    rng = S.PartitionRange(0, n, 0)
    for _ in range(3):
        S.select_by_threshold(acc, rng, 0.0258)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20):
        sel = S.select_by_threshold(acc, rng, 0.0258)
    b.record()
    torch.cuda.synchronize()
    us = a.elapsed_time(b) / 20 * 1e3
    k = sel.count()
    print(f"{dt}: select_by_threshold over {n} elements: {us:.1f} us/call, k = {k}, "
          f"{(n * acc.element_size() + k * (4 + acc.element_size())) / us / 1e3:.0f} GB/s algorithmic")
