#!/usr/bin/env python3
"""Benchmark: MiCRO sparsify + aggregate, µs per iteration on N B200s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c3]
    torchrun --nproc-per-node N bench.py --gpus N ...      (one process per GPU)
    python bench.py --impl reference ...                   (the reference's CPU code)

A step is one MiCRO iteration (harness.cpp:121-224) over one synthetic
gradient per worker: K1 (fused accumulate + select + compact + own-zero), the
exchange (N > 1), the ordered reduce, threshold update and the dense g/n.
Workload (default c3, BASELINE.json configs[2]): VGG-16-size n_g = 138M fp32,
d = 0.01, error feedback on, one worker per GPU (n = N).  Inputs are resident
in HBM (four pre-generated N(0,1) gradients, rotated) and 552 MB each, larger
than the 126 MB L2, so no flush is needed.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    "c3": dict(n_g=138_000_000, d=0.01, desc="VGG-16-size 138M fp32 gradient, d=0.01, EF on (BASELINE configs[2])"),
    "c1": dict(n_g=11_700_000, d=0.01, desc="ResNet-18-size 11.7M fp32 gradient, d=0.01 (BASELINE configs[0/1])"),
    "c4": dict(n_g=340_000_000, d=0.001, desc="BERT-large-size 340M fp32 gradient, d=0.001 (BASELINE configs[3])"),
    "c5_d001": dict(n_g=1_500_000_000, d=0.001, desc="GPT-2-XL-size 1.5B fp32 gradient, d=0.001 (configs[4])"),
    "c5_d01": dict(n_g=1_500_000_000, d=0.01, desc="GPT-2-XL-size 1.5B fp32 gradient, d=0.01 (configs[4])"),
    "c5_d1": dict(n_g=1_500_000_000, d=0.1, desc="GPT-2-XL-size 1.5B fp32 gradient, d=0.1 (configs[4])"),
}
# ALPHA: the controller's scaling factor.  The reference's default is 0.01
# (sparsifier.hpp:43), but at 0.01 its update settles into a period-2 cycle
# whose mean density sits ~8 % above d; the north star holds density within
# +-5 % of d, which the same controller meets at 0.001 at every BASELINE
# density (C3 +0.7 %, C1 +0.1 %, C4 d = 0.001 +2.4 %; 0.003 leaves C4 at
# +8.9 %: profiles/README.md).  Both arms run the same value (--alpha).
# From the warm start it adapts in ~1300 iterations at d = 0.01 and ~2500 at
# d = 0.001 (the residual's stationary spread is wider there): 3000 untimed ones.
ETA, ALPHA, SEED = 0.01, 0.001, 1
METRIC = "sparsify+aggregate µs/iter and select GB/s vs HBM peak at 1/2/4/8 B200"


def warm_delta0(d: float) -> float:
    """1 - d quantile of |eta*G| for G ~ N(0,1) (SURVEY.md §8d warm start)."""
    return statistics.NormalDist().inv_cdf(1 - d / 2) * ETA


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi-equivalent clocks/throttle reasons via NVML, sampled in a
    thread DURING the timed region."""
    NAMES = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
             0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks_setting"}

    def __init__(self, index: int):
        self.samples, self.reasons, self.ok = [], 0, False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max = None
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(0.001)

    def __enter__(self):
        if self.ok:
            self.th = threading.Thread(target=self._run, daemon=True)
            self.th.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.th.join()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml_unavailable"]}
        med = statistics.median(self.samples) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max, "samples": len(self.samples),
                "reasons": [v for k, v in self.NAMES.items() if self.reasons & k]}


# ---------------------------------------------------------------- reference


def host_info(threads: int) -> dict:
    """The host the CPU numbers were taken on."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"nproc": len(os.sched_getaffinity(0)), "cpu_model": model, "threads_used": threads}


def _fresh_normal(rng_pool, out: np.ndarray):
    """Fill `out` (float64) with fresh N(0,1) draws, one numpy Generator per
    host thread (they release the GIL), outside any timed region."""
    from concurrent.futures import ThreadPoolExecutor
    flat = out.reshape(-1)
    k = len(rng_pool)
    step = (flat.size + k - 1) // k
    with ThreadPoolExecutor(k) as ex:
        list(ex.map(lambda i: rng_pool[i].standard_normal(out=flat[i * step:(i + 1) * step]), range(k)))


def run_reference_converged(n_g: int, n: int, d: float, steps: int, warmup: int, adapt_iters: int = 1000,
                            adapt_n: int = 1 << 20, dense: bool = True, model: bool = True, threads: int = 1,
                            seed: int = SEED, grad32: bool = False):
    """The reference's own hot-path code (oracle/_ref: its sparsifier and
    collectives TUs compiled verbatim, re-driven in run_iteration's order),
    fp64, timed in the STATIONARY regime:

      1. adapt_iters iterations from the warm delta_0 at a sampled
         n_s = min(n_g, adapt_n) with fresh N(0,1) gradients (the threshold and
         residual reach their stationary law; both are scale-free in n_g);
      2. the converged state is transplanted into a full-size cluster: each
         worker's threshold, and its residual tiled to n_g (the coordinates
         are i.i.d. at stationarity, so the tiled residual has the stationary
         marginal law);
      3. `warmup` + `steps` iterations at the full n_g, a fresh gradient per
         step generated outside the timed region; each step is timed alone.

    grad32: every gradient is rounded to fp32 values first (BASELINE's "fp32
    gradient"), outside the timed region; the reference computes on them in
    fp64, as our f64 engine does on the same fp32 gradients.

    Returns per-step seconds, the realised density of each timed step, the
    first timed iteration and a description."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import RefCluster

    pool = [np.random.default_rng([seed, 7, i]) for i in range(max(1, min(16, len(os.sched_getaffinity(0)))))]
    delta0 = warm_delta0(d)
    n_s = min(n_g, max(adapt_n, n))
    small = RefCluster(n_s, n, density=d, delta0=delta0, alpha=ALPHA)
    small.set_options(dense=False, threads=threads)
    Gs = np.empty((n, n_s))
    def fresh(buf):
        _fresh_normal(pool, buf)
        if grad32:
            np.copyto(buf, buf.astype(np.float32))

    for t in range(adapt_iters):
        fresh(Gs)
        small.step(Gs, ETA, t)
    res = [small.residual(i) for i in range(n)]
    thr = np.empty(n)
    small.r.lib.ref_cluster_thresholds(small.h, thr)
    del small, Gs
    ref = RefCluster(n_g, n, density=d, delta0=delta0, alpha=ALPHA, model=model)
    ref.set_options(dense=dense, threads=threads)
    if n_s != n_g:
        for i in range(n):
            ref.set_state(i, np.resize(res[i], n_g), thr[i])
    else:
        for i in range(n):
            ref.set_state(i, res[i], thr[i])
    del res
    G = np.empty((n, n_g))
    times, dens = [], []
    t = adapt_iters
    for s in range(warmup + steps):
        fresh(G)
        t0 = time.perf_counter()
        r = ref.step(G, ETA, t)
        dt = time.perf_counter() - t0
        t += 1
        if s >= warmup:
            times.append(dt)
            dens.append(r["union_idx"].size / n_g)
    sample = (f"{steps} timed iterations (after {warmup} warm-up) at the full n_g={n_g}, n={n} workers "
              f"({'serially on 1 thread' if threads == 1 else f'per-worker loops on {threads} threads'}), fp64"
              f"{' on fp32-valued gradients' if grad32 else ''}, "
              f"the reference's sparsifier/collectives TUs compiled verbatim (oracle/_ref) driven in "
              f"run_iteration order with the model update{' and the dense all_reduce_sparse / n' if dense else ''}; "
              f"stationary start: {adapt_iters} adaptation iterations at n_s={n_s} (fresh N(0,1) gradients), "
              f"state transplanted (threshold; residual tiled to n_g); a fresh gradient per step")
    return dict(times=times, density=dens, first_timed_t=adapt_iters + warmup, sample=sample)


def reference_arm(args, wl):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    n = args.gpus
    threads = max(1, min(n, len(os.sched_getaffinity(0))))
    r = run_reference_converged(wl["n_g"], n, wl["d"], args.steps, args.warmup, adapt_iters=args.prime,
                                dense=args.dense, model=args.model, threads=threads, seed=args.seed,
                                grad32=args.grad == "f32" and args.sparsifier == "micro")
    per = statistics.mean(r["times"])
    us = per * 1e6
    dens = float(np.mean(r["density"]))
    line = {"metric": METRIC, "value": us, "unit": "us/iter", "n_gpus": n, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": per * 1e3, "higher_is_better": False, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": ("synthetic N(0,1) gradients rounded to fp32 values (numpy, fresh per step)" if args.grad == "f32"
                     else "synthetic N(0,1) gradients (numpy, fresh per step)"),
            "impl": "reference",
            "config": bench_config(args, wl, n),
            "protocol": {"adaptation_iterations": args.prime, "first_timed_t": r["first_timed_t"],
                         "median_us_per_step": float(np.median(r["times"])) * 1e6},
            "density": dens, "density_rel_err": dens / wl["d"] - 1.0,
            "host": host_info(threads),
            "cpu_baseline": {"value": us, "unit": "us/iter", "cores": threads, "kind": "reference",
                             "sample": r["sample"]},
            "e2e": {"value": us, "unit": "us/iter", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- our arm


def bench_config(args, wl, world: int) -> dict:
    """The workload both arms run (identical dicts: the ratio is like for like)."""
    W = args.cluster_workers if (world == 1 and args.cluster_workers > 1) else 1
    n = world * W
    label = wl["desc"]
    if args.workload == "c3" and n == 1:
        label = "C3 per-GPU slice (n=1): " + wl["desc"] + " — configs[2] runs n=8, one worker per GPU"
    return {"workload": label, "n_g": wl["n_g"], "density_target": wl["d"], "workers": n,
            "one_worker_per_gpu": W == 1, "eta": ETA, "alpha": ALPHA, "delta0": warm_delta0(wl["d"]),
            "error_feedback": True, "model_update": bool(args.model), "dense_g_over_n": bool(args.dense),
            "error_norm_recorded": bool(args.error_norm), "sparsifier": args.sparsifier,
            "arithmetic": "f64 (the reference's own, bit-exact with its code)" if args.dtype == "f64"
            else "f32 (the north star's gradient type)",
            "gradient": ("f32 (BASELINE configs' 'fp32 gradient'; widened exactly into the f64 state, so the "
                         "reference computes on the same values)"
                         if args.dtype == "f64" and args.grad == "f32" and args.sparsifier == "micro" else args.dtype),
            "parallelism": (f"dp{world} (exclusive cyclic partitions"
                            + (f", {args.transport} exchange)" if world > 1 else ")") if W == 1 else
                            f"{W} in-process workers on 1 GPU (exclusive cyclic partitions)"),
            "timing": "stationary regime: threshold and residual adapted before the timed steps; "
                      "a fresh N(0,1) gradient per step"}


def traffic_from_profiles(key: str):
    """DRAM bytes per launch of the dominant kernel from the ncu --set full
    capture of the same command (profiles/k1_dram_bytes.json)."""
    p = os.path.join(ROOT, "profiles", "k1_dram_bytes.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        v = j.get(key)
        if isinstance(v, dict):
            return v.get("bytes"), v.get("source")
        return v, "profiles/k1_dram_bytes.json"
    return None, None


def grad_dtype(args, tdt):
    """The gradients' element type: fp32 (BASELINE's "fp32 gradient"; widened
    exactly into the f64 state when the arithmetic is f64) or the arithmetic's."""
    import torch
    # (the comparison sparsifiers take gradients of their own dtype)
    return torch.float32 if args.grad == "f32" and args.sparsifier == "micro" else tdt


def device_measure(args, wl, tdt, dist, world, rank, local, dev, keep=False, gdt=None):
    """Adapt, warm up and time K steps of the device path at dtype tdt
    (gradients of dtype gdt, default grad_dtype(args, tdt)).
    Returns the measurement dict (and the engine + buffers when keep)."""
    import torch

    from paper_2310_00967_b200 import engine

    n_g, d = wl["n_g"], wl["d"]
    delta0 = warm_delta0(d)
    esz = 8 if tdt == torch.float64 else 4
    gdt = gdt or grad_dtype(args, tdt)
    gsz = 8 if gdt == torch.float64 else 4
    W = args.cluster_workers if (world == 1 and args.cluster_workers > 1) else 1
    if dist is not None:
        from paper_2310_00967_b200.dist import DistMicro
        m = DistMicro(n_g, transport=args.transport, density=d, initial_threshold=delta0, scaling_factor=ALPHA,
                      dense_output=args.dense, record_error_norm=args.error_norm, dtype=tdt, grad_dtype=gdt,
                      comm_device="cpu" if args.dist_backend == "gloo" else None)
    else:
        m = engine.Micro(n_g, W, density=d, initial_threshold=delta0, scaling_factor=ALPHA, dense_output=args.dense,
                         record_error_norm=args.error_norm, sparsifier=args.sparsifier, dtype=tdt,
                         grad_dtype=gdt)
    stream = torch.cuda.current_stream(dev)
    # the model update x -= g/n at the union is part of the reference's
    # iteration (harness.cpp:212-215)
    model = torch.zeros(n_g, device=dev, dtype=tdt)
    if args.model:
        m.set_model(model)

    # The threshold adapts for `prime` untimed iterations on fresh N(0,1)
    # gradients (generated between steps), reaching the stationary regime the
    # density target refers to.  The warm-up and timed steps
    # then read gradients already resident in HBM: one fresh buffer per step
    # when memory allows (same statistics as the prime phase), otherwise R
    # buffers rotated.
    t = 0
    gen = [torch.empty(n_g, device=dev, dtype=gdt) for _ in range(W)]
    for _ in range(args.prime):
        for i in range(W):
            engine.synth_gaussian(gen[i], args.seed, rank + i, t)
        m.step(gen, ETA, t)
        t += 1
    del gen
    torch.cuda.synchronize()
    need = (args.warmup + args.steps) * W
    R = max(W + 1, min(need, args.buffers, int(0.5 * torch.cuda.mem_get_info(dev)[0] // (gsz * n_g))))
    G = [torch.empty(n_g, device=dev, dtype=gdt) for _ in range(R)]
    for r in range(R):
        engine.synth_gaussian(G[r], args.seed, rank + r % W, t + r)
    t0_bufs = t
    # not enough HBM for one resident gradient per step (C5 in f64: 12 GB
    # each): each step's gradients are generated fresh into the R buffers
    # just before the step, outside its events (re-fed gradients would make
    # the residual grow coherently and inflate the selection)
    fresh = R < need

    def grads(t):
        q = (t - t0_bufs) * W
        out = [G[(q + i) % R] for i in range(W)]
        if fresh:
            for i, g in enumerate(out):
                engine.synth_gaussian(g, args.seed, rank + i, t)
        return out

    for s in range(args.warmup):
        m.step(grads(t), ETA, t)
        t += 1
    torch.cuda.synchronize()

    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    t_first = t
    # CUDA events around K1's streaming pass, inside the library, on every
    # 4th step of the timed region (sampled, so the step time stays the step's)
    m.kernel_timing(True, every=4)
    if dist:
        m.exchange_timing(True)
    # the step's working set (e, G, x) fits in L2 at the small workloads:
    # there, flush L2 between timed steps, outside the per-step event windows:
    # a 256 MB write (evicts the step's lines) then a 256 MB read (so the
    # flush's own dirty lines are written back inside the flush, not charged
    # to the next step).  At C3 and up the inputs are larger than L2.
    flush = args.flush_l2 == "on" or (args.flush_l2 == "auto" and (2 * esz + gsz) * n_g < 2 * 126e6)
    scratch = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if flush else None
    scratch2 = torch.empty(64 << 20, dtype=torch.float32, device=dev) if flush else None
    per_step = flush or fresh  # each step timed alone (events around the step only)
    step_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)] if per_step else []
    with ClockSampler(local) as clk:
        start.record(stream)
        for s in range(args.steps):
            gs = grads(t)  # fresh mode: generated here, before the step's events
            if flush:
                scratch.fill_(s & 0xFF)
                scratch2.sum()
            if per_step:
                step_ev[s][0].record(stream)
            m.step(gs, ETA, t)  # the whole iteration, one library call
            if per_step:
                step_ev[s][1].record(stream)
            t += 1
        end.record(stream)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in step_ev]
    # the every-4th step carrying K1's event pair (k1a below) pays for it: the
    # events break the PDL chain between k1_stream and k1_gather (~7 us at C1).
    # With per-step events (flush mode) the step time is taken over the other
    # steps; without them (C3 and up) the sampled steps stay in (< 1 %).
    plain = [v for s_, v in enumerate(step_ms) if s_ % 4] or step_ms
    total_ms = statistics.mean(plain) * args.steps if per_step else start.elapsed_time(end)
    k1a_ms = [float(v) for v in m.kernel_times(args.steps)]  # k1_stream alone (sampled launches)
    m.kernel_timing(False)
    xchg_ms = None
    cdev = dev if args.dist_backend == "nccl" else "cpu"
    if dist:
        xt = m.exchange_times()
        m.exchange_timing(False)
        v = torch.tensor([statistics.mean(xt) if xt else 0.0], device=cdev, dtype=torch.float64)
        dist.all_reduce(v, op=dist.ReduceOp.MAX)
        xchg_ms = float(v[0])
        v = torch.tensor([total_ms], device=cdev, dtype=torch.float64)
        dist.all_reduce(v, op=dist.ReduceOp.MAX)
        total_ms = float(v[0])
    ms_step = total_ms / args.steps
    hist = m.history(args.steps)
    K = hist["K"].astype(np.float64)
    k_own = hist["counts"][:, 0].astype(np.float64)
    out = dict(ms_step=ms_step, step_ms=step_ms, k1a_ms=k1a_ms, xchg_ms=xchg_ms, K=K, k_own=k_own, R=R,
               flush=flush, fresh=fresh, t_first=t_first, t_next=t, W=W, esz=esz, gsz=gsz, clocks=clk.summary(),
               transport=getattr(m, "transport", None))
    if keep:
        out.update(m=m, G=G)
    else:
        m.close()
        del G
        torch.cuda.empty_cache()
    return out


def roofline_of(args, r, wl, world, peak, peak_kind):
    """Algorithmic bytes of the dominant kernel (k1_stream) and of the step."""
    n_g, W, esz, gsz = wl["n_g"], r["W"], r["esz"], r["gsz"]
    K, k_own = r["K"], r["k_own"]
    # k1_stream: read e and G, write e (all n_g) + one (int32,
    # value) pair per selection; with the dense g/n (fused at n = 1) the
    # current union's values and the previous union's zeros (2 values per
    # entry).  top-k's compaction reads acc only (the histogram passes formed
    # it); CLT-k's leader is top-k, its other workers select by threshold.
    acc_only = {"topk": W, "cltk": 1}.get(args.sparsifier, 0)
    # one worker selecting: the union is its selection and K1 maintains the
    # dense g/n (every sparsifier but the dense baseline's one-pass kernel)
    dense_fused = args.dense and world == 1 and W == 1 and args.sparsifier != "dense"
    k1_bytes = ((n_g * (esz * acc_only + (2.0 * esz + gsz) * (W - acc_only)) / W) + (4.0 + esz) * float(k_own.mean())
                + (2.0 * esz * float(K.mean()) if dense_fused else 0.0))
    k1a_avg_ms = statistics.mean(r["k1a_ms"]) if r["k1a_ms"] else r["ms_step"]
    achieved = k1_bytes / (k1a_avg_ms * 1e-3) / 1e9
    # whole step vs the same roofline: K1 + the union (8 B at n = 1: written by
    # the gather) + the model's read-modify-write (2 values per union entry) +
    # the dense g/n when not fused + the cluster reduce (W reads + zeroing)
    extras = ((4.0 + esz) * float(K.mean())
              + (2.0 * esz * float(K.mean()) if args.model else 0.0)
              + (2.0 * esz * float(K.mean()) if (args.dense and not dense_fused) else 0.0)
              + (2.0 * esz * float(K.mean()) * W if W > 1 else 0.0))
    if acc_only:
        # top-k is an exact radix select: pass 1 forms acc (e, G read, acc
        # written), one acc-only pass per further 11-bit digit, the tie count
        # and the compaction; CLT-k's other workers accumulate only
        digits = -(-8 * esz // 11)
        per_topk = (n_g * (3.0 * esz + esz * (digits - 1) + 2.0 * esz) + (4.0 + esz) * float(k_own.mean())
                    + (2.0 * esz * float(K.mean()) if dense_fused else 0.0))
        step_bytes = acc_only * per_topk + (W - acc_only) * 3.0 * esz * n_g + extras
    else:
        step_bytes = W * k1_bytes + extras
    return {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "kernel": "k1_stream", "algorithmic_bytes_per_launch": k1_bytes, "avg_launch_ms": k1a_avg_ms,
            "peak_source": peak_kind,
            "timed_launches": f"{len(r['k1a_ms'])} of {args.steps} (every 4th, CUDA events on the launch stream)",
            "step_frac": step_bytes / (r["ms_step"] * 1e-3) / 1e9 / peak}


def our_arm(args, wl):
    import torch

    from paper_2310_00967_b200 import engine

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if args.dist_backend == "gloo":  # code-path check of N > 1 on one GPU: ranks share it, numbers are not valid
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    n_g, d = wl["n_g"], wl["d"]
    tdt = torch.float64 if args.dtype == "f64" else torch.float32
    dist = None
    if world > 1:
        import torch.distributed as tdist
        if args.dist_backend == "gloo":
            tdist.init_process_group("gloo")
        else:
            tdist.init_process_group("nccl", device_id=dev)
        dist = tdist
    r = device_measure(args, wl, tdt, dist, world, rank, local, dev, keep=True)
    m, G, W, esz, gsz = r["m"], r["G"], r["W"], r["esz"], r["gsz"]
    gdt = grad_dtype(args, tdt)
    t = r["t_next"]
    ms_step, K, k_own = r["ms_step"], r["K"], r["k_own"]
    density = float(K.mean() / n_g)
    peak, peak_kind = peaks()
    roof = roofline_of(args, r, wl, world, peak, peak_kind)
    tkey = f"{args.workload}_{args.dtype}{'_g32' if gsz != esz else ''}{'_dense' if args.dense else ''}"
    roof["traffic"], roof["traffic_source"] = traffic_from_profiles(tkey)
    # our kernels per step: k1_stream, k1_gather (+ threshold update + model
    # update + dense g/n) at n = 1; a W-worker cluster: 2 per worker +
    # k_cluster_reduce + k_finalize (+ k_dense_clear); n > 1 ranks: K1 x2 +
    # the exchange + finalize (NCCL kernels not counted)
    launches_per_step = ((2 if W == 1 else 2 * W + 2 + (1 if args.dense else 0)) if world == 1
                         else {"peer": 5, "peer_pull": 4, "nccl": 6, "abi_peer": 5, "abi_nccl": 6}[r["transport"]]
                         + (1 if args.dense else 0))  # + k_dense_clear (aux stream) at n > 1
    if args.sparsifier != "micro":  # baselines.cuh: per selecting worker, top-k = init + 2 per digit +
        # tie count/find + stream + gather (fp32: 11), hard = 2, else accumulate + count = 2; then
        # union marks (W) + 3 scan passes + emit + reduce + finalize (dense: dense_all + finalize)
        per = {"topk": 11 * W, "cltk": 11 + 2 * (W - 1), "hard": 2 * W, "dense": 2 * W}[args.sparsifier]
        # one worker (not dense): the selection is the union, the gather finalizes
        launches_per_step = per + (2 if args.sparsifier == "dense" else 0 if W == 1 else W + 6)

    # ---- end to end through the public API with host buffers ----
    cdev = dev if args.dist_backend == "nccl" else "cpu"
    if world == 1:
        # one distinct pinned host gradient per e2e step (the same statistics
        # as the timed steps; re-feeding one gradient would make the residual
        # grow coherently and inflate the selection)
        ke = max(3, min(args.steps, 10))
        nb = int(max(2, min(ke + 1, 16e9 // (gsz * n_g * W))))  # <= 16 GB of pinned host gradients
        hGs = []
        for b in range(nb):
            hG = torch.empty(W * n_g, dtype=gdt).pin_memory()
            for i in range(W):
                engine.synth_gaussian(G[i], args.seed, rank + i, t + 1 + b)  # fresh: steps t+1 .. t+nb
                hG[i * n_g:(i + 1) * n_g].copy_(G[i].cpu())
            hGs.append(hG)
        idx = torch.empty(n_g, dtype=torch.int32).pin_memory().numpy()  # pinned result buffers
        sums = torch.empty(n_g, dtype=tdt).pin_memory().numpy()
        m.step_host(hGs[-1], ETA, t, idx, sums)  # warm (staging allocation); its gradient is not reused
        t += 1
        kk = []
        t0 = time.perf_counter()
        per = []
        for s in range(ke):
            ts = time.perf_counter()
            i_, _s = m.step_host(hGs[s % (nb - 1)], ETA, t, idx, sums)  # returns after the D2H landed
            per.append(time.perf_counter() - ts)
            kk.append(i_.size)
            t += 1
        e2e_s = (time.perf_counter() - t0) / ke
        e2e = {"value": e2e_s * 1e6, "unit": "us/iter", "h2d_bytes_per_step": gsz * n_g * W,
               "median_us_per_step": statistics.median(per) * 1e6, "min_us_per_step": min(per) * 1e6,
               "d2h_bytes_per_step": int((4 + esz) * statistics.mean(kk) + 8 + 4),
               "api": "micro_step_host (include/micro.h)",
               "host_gradients": f"{nb - 1} distinct pinned buffers over {ke} steps",
               "density": float(statistics.mean(kk)) / n_g,
               # what bounds it: the H2D of the gradient over PCIe (Gen5 x16: ~64 GB/s nominal)
               "h2d_gbs_effective": gsz * n_g * W / e2e_s / 1e9}
        del hGs
    else:
        # N ranks: each copies its own pinned host gradient in, steps through
        # DistMicro, and reads the union back; the max over ranks is reported
        ke = max(3, min(args.steps, 10))
        nb = int(max(2, min(ke + 1, 4e9 // (gsz * n_g))))
        hGs = []
        for b in range(nb):
            engine.synth_gaussian(G[0], args.seed, rank, t + 1 + b)
            hGs.append(G[0].cpu().pin_memory())
        dG = torch.empty(n_g, device=dev, dtype=gdt)
        idx = torch.empty(n_g, dtype=torch.int32).pin_memory().numpy()
        sums = torch.empty(n_g, dtype=tdt).pin_memory().numpy()
        dG.copy_(hGs[-1], non_blocking=True)
        m.step([dG], ETA, t)
        m.union(idx, sums)
        t += 1
        kk = []
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for s in range(ke):
            dG.copy_(hGs[s % (nb - 1)], non_blocking=True)
            m.step([dG], ETA, t)
            i_, _s = m.union(idx, sums)
            kk.append(i_.size)
            t += 1
        torch.cuda.synchronize()
        v = torch.tensor([(time.perf_counter() - t0) / ke], device=cdev, dtype=torch.float64)
        dist.all_reduce(v, op=dist.ReduceOp.MAX)
        e2e = {"value": float(v[0]) * 1e6, "unit": "us/iter", "h2d_bytes_per_step": gsz * n_g,
               "d2h_bytes_per_step": int((4 + esz) * statistics.mean(kk) + 8 + 4),
               "api": "DistMicro.step + union (paper_2310_00967_b200/dist.py)",
               "host_gradients": f"{nb - 1} distinct pinned buffers per rank over {ke} steps",
               "density": float(statistics.mean(kk)) / n_g, "per": "rank (max over ranks)"}
        del hGs
    m.close()
    del G, m
    torch.cuda.empty_cache()

    # ---- the same measurement in the other arithmetic (N = 1, MiCRO) ----
    other = None
    if world == 1 and args.sparsifier == "micro" and not args.no_other_dtype:
        otdt = torch.float32 if tdt == torch.float64 else torch.float64
        ro = device_measure(args, wl, otdt, None, world, rank, local, dev)
        rf = roofline_of(args, ro, wl, world, peak, peak_kind)
        other = {"dtype": "f32" if otdt == torch.float32 else "f64", "value": ro["ms_step"] * 1e3,
                 "unit": "us/iter", "density": float(ro["K"].mean() / n_g),
                 "roofline": {k: rf[k] for k in ("achieved", "peak", "frac", "algorithmic_bytes_per_launch",
                                                 "avg_launch_ms", "step_frac")}}
    # ---- f64 arithmetic on f64 gradients (the reference's own input type) ----
    other_grad = None
    if (world == 1 and args.sparsifier == "micro" and not args.no_other_dtype and tdt == torch.float64
            and gsz != esz):
        ro = device_measure(args, wl, tdt, None, world, rank, local, dev, gdt=torch.float64)
        rf = roofline_of(args, ro, wl, world, peak, peak_kind)
        other_grad = {"dtype": "f64", "gradient": "f64", "value": ro["ms_step"] * 1e3, "unit": "us/iter",
                      "density": float(ro["K"].mean() / n_g),
                      "roofline": {k: rf[k] for k in ("achieved", "peak", "frac", "algorithmic_bytes_per_launch",
                                                      "avg_launch_ms", "step_frac")}}

    # ---- CPU baseline: the reference's own code on this host (rank 0, N = 1) ----
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            cr = run_reference_converged(n_g, W, d, steps=args.cpu_steps, warmup=1, adapt_iters=args.prime,
                                         dense=args.dense, model=args.model, threads=1, seed=args.seed,
                                         grad32=gsz == 4)
            cd = float(np.mean(cr["density"]))
            cpu = {"value": statistics.mean(cr["times"]) * 1e6, "unit": "us/iter", "cores": 1, "kind": "reference",
                   "sample": cr["sample"], "density": cd, "first_timed_t": cr["first_timed_t"],
                   "density_vs_ours": cd / density - 1.0, "host": host_info(1)}
        except Exception as ex:  # the checker is optional at run time; the GPU number stands
            cpu = {"value": None, "unit": "us/iter", "cores": 1, "kind": "reference", "sample": f"failed: {ex}"}

    # the exchange against the NVLink roofline (N > 1): bytes received per GPU,
    # 4(K-k) foreign indices + 4k(n-1) contributions + 4(K-k) sums
    exchange_line = None
    if dist and r["xchg_ms"]:
        Km, km = float(K.mean()), float(k_own.mean())
        b_net = 4.0 * (Km - km) + 4.0 * km * (world - 1) + 4.0 * (Km - km)
        xms = r["xchg_ms"]
        exchange_line = {"bound": "nvlink", "achieved": b_net / (xms * 1e-3) / 1e9, "peak": 900.0,
                         "unit": "GB/s", "frac": b_net / (xms * 1e-3) / 1e9 / 900.0,
                         "bytes_per_gpu": b_net, "avg_ms": xms, "transport": r["transport"],
                         "peak_source": "NVLink 5 per direction per GPU (nominal)",
                         "timed": "exchange kernels, barriers excluded" if r["transport"] != "nccl"
                         else "the whole NCCL protocol"}

    if rank == 0:
        R = r["R"]
        line = {
            "metric": METRIC, "value": ms_step * 1e3, "unit": "us/iter", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": False, "scaling": "weak",
            "vs_baseline": None, "dtype": args.dtype,
            "data": f"synthetic N(0,1) {'f32' if gsz == 4 else 'f64'} gradients (include/micro_synth.h)",
            "config": bench_config(args, wl, world),
            "protocol": {"adaptation_iterations": args.prime, "first_timed_t": r["t_first"], "seed": args.seed,
                         "inputs": (f"{R} resident N(0,1) gradient buffers ("
                                    + ("one fresh gradient per step" if not r["fresh"] else
                                       "each step's gradient generated fresh into them just before the step, "
                                       "outside its events; steps timed one by one")
                                    + (f"); L2 flushed between timed steps (256 MB write + 256 MB read outside "
                                       f"the per-step events: the working set {(2 * esz + gsz) * n_g / 1e6:.0f} MB "
                                       f"would fit L2)" if r["flush"] else f"); each {gsz}*n_g bytes > L2 (no flush "
                                       f"needed)" if gsz * n_g > 126e6 else "); L2 NOT flushed (--flush-l2 off)")),
                         "median_us_per_step": (float(np.median(r["step_ms"])) * 1e3 if r["step_ms"] else None)},
            "density": density, "density_rel_err": density / d - 1.0,
            "density_reference": (cpu or {}).get("density"),
            "density_window": {"first_quarter": float(K[: max(1, len(K) // 4)].mean() / n_g),
                               "last_quarter": float(K[-max(1, len(K) // 4):].mean() / n_g),
                               "median": float(np.median(K) / n_g)},
            "select_gbs": roof["achieved"],
            "roofline": roof,
            "exchange": exchange_line,
            "other_dtype": other,
            "other_gradient": other_grad,
            "clocks": r["clocks"],
            "gpu_launches": launches_per_step * args.steps,
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


def main():
    global ALPHA
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="c3")
    ap.add_argument("--prime", type=int, default=3000, help="untimed threshold-adaptation iterations")
    ap.add_argument("--buffers", type=int, default=256, help="max resident gradient buffers")
    ap.add_argument("--cpu-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--grad", choices=["f32", "same"], default="f32",
                    help="gradient element type: f32 (BASELINE's fp32 gradient; widened exactly into f64 state "
                         "with --dtype f64) or the arithmetic's own")
    ap.add_argument("--no-dense", dest="dense", action="store_false",
                    help="skip the dense averaged gradient g/n (all_reduce_sparse / n, collectives.cpp:51-57)")
    ap.add_argument("--cluster-workers", type=int, default=1,
                    help="N = 1 only: W in-process workers on the GPU (the reference's in-process cluster)")
    ap.add_argument("--no-model", dest="model", action="store_false", help="skip the model update x -= g/n")
    ap.add_argument("--sparsifier", choices=["micro", "topk", "cltk", "hard", "dense"], default="micro",
                    help="N = 1: a comparison sparsifier of the reference's harness instead of MiCRO")
    ap.add_argument("--dist-backend", choices=["nccl", "gloo"], default="nccl",
                    help="gloo: exercise the N > 1 path with all ranks on one GPU (code check only)")
    ap.add_argument("--transport", choices=["peer", "peer_pull", "nccl", "abi_peer", "abi_nccl"], default="peer",
                    help="N > 1: exchange over peer memory (bulk or pull) or the collective protocol, driven from "
                         "Python over torch.distributed, or entirely inside the library (abi_*: "
                         "micro_dist_init_nccl + micro_step, what a C++ host calls)")
    ap.add_argument("--seed", type=int, default=SEED, help="synthetic gradient stream (SURVEY.md 8d: 1, 2, 3)")
    ap.add_argument("--flush-l2", choices=["auto", "on", "off"], default="auto",
                    help="flush L2 between timed steps (auto: when e, G and x would fit in L2)")
    ap.add_argument("--dtype", choices=["f32", "f64"], default="f64",
                    help="f64 (default): the reference's own arithmetic (bit-exact with its code); f32: the "
                         "north star's gradient type (reported beside the f64 line as other_dtype)")
    ap.add_argument("--no-other-dtype", action="store_true", help="skip the other-dtype measurement")
    ap.add_argument("--error-norm", action="store_true",
                    help="also record the per-step error norm ||e_{t+1}|| (fused into k1_stream); off by "
                         "default, like the reference arm's timed step")
    ap.add_argument("--alpha", type=float, default=ALPHA,
                    help="the threshold controller's scaling factor, both arms (sparsifier.hpp:43: the "
                         "reference's default is 0.01, +8 %% density; 0.001 holds d within +-5 %%)")
    args = ap.parse_args()
    ALPHA = args.alpha
    wl = WORKLOADS[args.workload]
    if args.impl == "reference":
        return reference_arm(args, wl)
    return our_arm(args, wl)


if __name__ == "__main__":
    sys.exit(main())
