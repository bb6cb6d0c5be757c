"""Where does the small-config (C1) step time go?  Times the same converged
MiCRO step (11.7M fp32, d = 0.01, n = 1, model update) under different
cache states and timing methods (CUDA events only).

    python tools/c1_exp.py [--dense]
"""
import argparse
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2310_00967_b200 import engine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dense", action="store_true")
ap.add_argument("--n-g", type=int, default=11_700_000)
ap.add_argument("--dtype", default="f32")
a = ap.parse_args()
n_g = a.n_g
tdt = torch.float64 if a.dtype == "f64" else torch.float32
m = engine.Micro(n_g, 1, density=0.01, initial_threshold=0.02576, dense_output=a.dense, dtype=tdt)
x = torch.zeros(n_g, device="cuda", dtype=tdt)
m.set_model(x)
R = 64
G = [torch.empty(n_g, device="cuda", dtype=tdt) for _ in range(R)]
for i, g in enumerate(G):
    engine.synth_gaussian(g, 1, 0, i)
t = 0
for _ in range(600):
    m.step([G[t % R]], 0.01, t)
    t += 1
torch.cuda.synchronize()
w = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
r = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
r2 = torch.empty(128 << 20, dtype=torch.float32, device="cuda")


def ev():
    return torch.cuda.Event(enable_timing=True)


def loop(n, flush=None, per_step=False, step=True):
    global t
    s0, s1 = ev(), ev()
    per = []
    s0.record()
    for _ in range(n):
        if flush:
            flush()
        if per_step:
            e0, e1 = ev(), ev()
            e0.record()
        if step:
            m.step([G[t % R]], 0.01, t)
            t += 1
        if per_step:
            e1.record()
            per.append((e0, e1))
    s1.record()
    torch.cuda.synchronize()
    tot = s0.elapsed_time(s1) * 1e3 / n
    ps = statistics.median([p.elapsed_time(q) * 1e3 for p, q in per]) if per else None
    return tot, ps


res = {}
res["back_to_back"] = loop(200)[0]
fl = {"fill": lambda: w.fill_(1), "fill+sum": lambda: (w.fill_(1), r.sum()), "sum512": lambda: r2.sum()}
for k, f in fl.items():
    both = loop(100, flush=f)[0]
    only = loop(100, flush=f, step=False)[0]
    res[f"{k}: total-minus-flush"] = both - only
    res[f"{k}: per-step events (median)"] = loop(100, flush=f, per_step=True)[1]
m.kernel_timing(True, every=1)
res["fill+sum: per-step events, k1 timing on"] = loop(100, flush=fl["fill+sum"], per_step=True)[1]
k1 = m.kernel_times(100)
res["k1_stream event time (median)"] = float(statistics.median(k1)) * 1e3
m.kernel_timing(False)
print(f"n_g={n_g} {a.dtype} dense={a.dense}")
for k, v in res.items():
    print(f"  {k:45s} {v:8.1f} us")
