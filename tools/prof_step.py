"""Profiling driver: adapt a workload to its stationary regime, then run a few
steps between cudaProfilerStart/Stop so `ncu --profile-from-start off`
captures exactly those steps' kernels.

    python tools/prof_step.py --workload c3 --dtype f64 [--dense] [--mode single|cluster|group] [--n 8]
    ncu --profile-from-start off --set full ... python tools/prof_step.py ...

Without ncu it prints CUDA-event times per step (a sanity check that the
profiled command is the bench's step)."""
import argparse
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import ALPHA, ETA, WORKLOADS, warm_delta0  # noqa: E402
from paper_2310_00967_b200 import engine  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c3", choices=sorted(WORKLOADS))
    ap.add_argument("--dtype", default="f32", choices=["f32", "f64"])
    ap.add_argument("--dense", action="store_true")
    ap.add_argument("--grad", default="same", choices=["same", "f32"], help="f32: fp32 gradients (f64 state)")
    ap.add_argument("--error-norm", action="store_true", help="record the error norm (bench.py: off by default)")
    ap.add_argument("--no-model", dest="model", action="store_false")
    ap.add_argument("--mode", default="single", choices=["single", "cluster", "group"])
    ap.add_argument("--n", type=int, default=1)
    ap.add_argument("--prime", type=int, default=3000)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--flush", action="store_true", help="flush L2 between profiled steps")
    a = ap.parse_args()
    wl = WORKLOADS[a.workload]
    n_g, d = wl["n_g"], wl["d"]
    tdt = torch.float64 if a.dtype == "f64" else torch.float32
    gdt = torch.float32 if a.grad == "f32" else tdt
    kw = dict(density=d, initial_threshold=warm_delta0(d), scaling_factor=ALPHA, dense_output=a.dense, dtype=tdt,
              grad_dtype=gdt, record_error_norm=a.error_norm)
    n = a.n if a.mode != "single" else 1
    if a.mode == "group":
        from paper_2310_00967_b200.dist import GroupMicro
        g = GroupMicro(n_g, n, devices=[0] * n, **kw)
        step = g.step
        xs = [torch.zeros(n_g, dtype=tdt, device="cuda") for _ in range(n)]
        if a.model:
            for m, x in zip(g.ranks, xs):
                m.set_model(x)
    else:
        m = engine.Micro(n_g, n, **kw)
        step = m.step
        x = torch.zeros(n_g, dtype=tdt, device="cuda")
        if a.model:
            m.set_model(x)
    G = [torch.empty(n_g, dtype=gdt, device="cuda") for _ in range(n)]
    t = 0
    for _ in range(a.prime):
        for i in range(n):
            engine.synth_gaussian(G[i], 1, i, t)
        step(G, ETA, t)
        t += 1
    torch.cuda.synchronize()
    scratch = torch.empty(256 << 20, dtype=torch.uint8, device="cuda") if a.flush else None
    scratch2 = torch.empty(64 << 20, dtype=torch.float32, device="cuda") if a.flush else None
    times = []
    torch.cuda.cudart().cudaProfilerStart()
    for _ in range(a.steps):
        for i in range(n):
            engine.synth_gaussian(G[i], 1, i, t)
        if a.flush:
            scratch.fill_(t & 0xFF)
            scratch2.sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        step(G, ETA, t)
        if a.mode == "group":
            for s in g.streams:
                torch.cuda.current_stream().wait_stream(s)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) * 1e3)
        t += 1
    torch.cuda.cudart().cudaProfilerStop()
    print(f"{a.workload} {a.dtype} mode={a.mode} n={n} dense={a.dense}: step us {[round(v, 1) for v in times]}, "
          f"median {statistics.median(times):.1f}")


if __name__ == "__main__":
    main()
