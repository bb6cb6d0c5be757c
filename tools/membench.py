"""HBM reference points for the K1 access pattern (12 B/element: read e and
G, write e) on this B200, next to K1 itself.  CUDA-event timed, best of N.

    python tools/membench.py [n_g]
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) * 1e-3)
    return best


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 138_000_000
    e = torch.randn(n, device="cuda")
    g = torch.randn(n, device="cuda")
    out = {}
    t = timeit(lambda: e.copy_(g))
    out["copy (1R:1W, 8 B/elem)"] = 8 * n / t / 1e9
    t = timeit(lambda: e.add_(g, alpha=0.01))
    out["torch add_ e += a*G (2R:1W, 12 B/elem)"] = 12 * n / t / 1e9
    t = timeit(lambda: torch.add(e, g, alpha=0.01, out=e))
    out["torch add out=e (12 B/elem)"] = 12 * n / t / 1e9
    t = timeit(lambda: torch.sum(e))
    out["sum (read only, 4 B/elem)"] = 4 * n / t / 1e9
    from paper_2310_00967_b200 import engine
    for cfg in ("k1",):
        m = engine.Micro(n, 1, initial_threshold=0.03)
        state = {"t": 0}

        def step():
            m.compress([g], 0.01, state["t"])
            m.aggregate()
            state["t"] += 1
        for _ in range(50):
            step()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        times = []
        for _ in range(20):
            a.record()
            m.compress([g], 0.01, state["t"])
            b.record()
            m.aggregate()
            state["t"] += 1
            torch.cuda.synchronize()
            times.append(a.elapsed_time(b) * 1e-3)
        k = m.query().K
        out["K1 (12 B/elem + pairs)"] = (12 * n + 8 * k) / min(times) / 1e9
        m.close()
    print(json.dumps({k: round(v, 1) for k, v in out.items()}, indent=1))


if __name__ == "__main__":
    main()
