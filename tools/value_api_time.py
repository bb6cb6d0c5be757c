"""Per-call time of every value-level drop-in function (sparsim.py, the
reference's sparsim:: free functions on device arrays) at C3 size, n = 8
workers for the collectives: the run_iteration order built from the value
calls.  CUDA events around `reps` calls each (Python face: outputs allocated
by torch's caching allocator, counts read back where the call returns them)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_00967_b200 import sparsim as S  # noqa: E402

n_g, n, d, reps = 138_000_000, 8, 0.01, 10
dt = torch.float32 if len(sys.argv) > 1 and sys.argv[1] == "f32" else torch.float64


def timed(name, fn):
    for _ in range(2):
        out = fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        out = fn()
    b.record()
    torch.cuda.synchronize()
    print(f"{name:34s} {a.elapsed_time(b) / reps * 1e3:10.1f} us/call", flush=True)
    return out


e = torch.randn(n_g, device="cuda", dtype=dt) * 0.01
g = torch.randn(n_g, device="cuda", dtype=dt)
acc = timed("accumulate (n_g)", lambda: S.accumulate(e, 0.01, g))
thr = 2.576 * 0.01
sel = timed("select_by_threshold (n_g/n range)", lambda: S.select_by_threshold(acc, S.partition(n_g, n, 0, 0), thr))
timed("select_topk (n_g, k = d*n_g)", lambda: S.select_topk(acc, S.PartitionRange(0, n_g, 0), int(d * n_g)))
timed("hard_threshold_select (n_g)", lambda: S.hard_threshold_select(acc, thr))
accs = [acc] + [torch.randn(n_g, device="cuda", dtype=dt) * 0.01 for _ in range(n - 1)]
sels = [S.select_by_threshold(accs[i], S.partition(n_g, n, 0, i), thr) for i in range(n)]
agg = timed("all_gather_indices (n = 8)", lambda: S.all_gather_indices(sels))
print(f"  K = {agg.indices.numel()}")
timed("all_reduce_sparse_values (n = 8)", lambda: S.all_reduce_sparse_values(accs, agg))
timed("all_reduce_sparse (dense, n = 8)", lambda: S.all_reduce_sparse(accs, agg))
timed("compensate (K indices)", lambda: S.compensate(acc.clone(), agg.indices))
timed("error_metric (n = 8)", lambda: S.error_metric(accs))
