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
ETA, ALPHA, SEED = 0.01, 0.01, 1
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


def traffic_from_profiles(workload: str):
    p = os.path.join(ROOT, "profiles", "k1_dram_bytes.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return j.get(workload)
    return None


# ---------------------------------------------------------------- reference


def run_reference_cluster(n_g: int, n: int, d: float, steps: int, warmup: int, seed: int = SEED):
    """The reference's own hot-path code (oracle/_ref) driven in run_iteration
    order: fp64, one host thread, all n workers serially.  Returns per-step
    seconds."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import RefCluster

    rng = np.random.default_rng(seed)
    ref = RefCluster(n_g, n, density=d, delta0=warm_delta0(d), alpha=ALPHA)
    G = [rng.standard_normal((n, n_g)) for _ in range(2)]
    times = []
    for s in range(warmup + steps):
        t0 = time.perf_counter()
        ref.step(G[s % 2], ETA, s)
        dt = time.perf_counter() - t0
        if s >= warmup:
            times.append(dt)
    del ref, G
    return times


def reference_arm(args, wl):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    n = args.gpus
    n_g = wl["n_g"]
    # bounded sample: keep (warmup + steps) * n * n_g * ~8 ns under ~150 s
    frac = min(1.0, 150.0 / max(1e-9, (args.warmup + args.steps) * n * n_g * 8e-9))
    n_s = max(n * 1024, int(n_g * frac))
    times = run_reference_cluster(n_s, n, wl["d"], args.steps, args.warmup)
    per = statistics.mean(times) * (n_g / n_s)
    us = per * 1e6
    sample = (f"{args.steps} timed iterations (after {args.warmup} warm-up) of the reference's MiCRO iteration "
              f"(sparsifier/collectives TUs compiled verbatim, fp64, n={n} workers serially on 1 thread) at "
              f"n_g={n_s}" + (f", scaled x{n_g / n_s:.2f} to n_g={n_g}" if n_s != n_g else ""))
    line = {"metric": METRIC, "value": us, "unit": "us/iter", "n_gpus": n, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": per * 1e3, "higher_is_better": False, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic N(0,1) gradients",
            "impl": "reference",
            "config": {"workload": wl["desc"], "n_g": n_g, "density": wl["d"], "workers": n},
            "cpu_baseline": {"value": us, "unit": "us/iter", "cores": 1, "kind": "reference", "sample": sample},
            "e2e": {"value": us, "unit": "us/iter", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- our arm


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
    delta0 = warm_delta0(d)
    tdt = torch.float64 if args.dtype == "f64" else torch.float32
    esz = 8 if args.dtype == "f64" else 4
    # W workers per process: 1 (one per GPU), or --cluster-workers W at N = 1:
    # the reference's own in-process cluster (harness.cpp:121-224) on one GPU
    W = args.cluster_workers if (world == 1 and args.cluster_workers > 1) else 1
    dist = None
    if world > 1:
        import torch.distributed as tdist

        from paper_2310_00967_b200.dist import DistMicro
        if args.dist_backend == "gloo":
            tdist.init_process_group("gloo")
        else:
            tdist.init_process_group("nccl", device_id=dev)
        dist = tdist
        m = DistMicro(n_g, transport=args.transport, density=d, initial_threshold=delta0, scaling_factor=ALPHA,
                      dense_output=args.dense, record_error_norm=args.error_norm, dtype=tdt,
                      comm_device="cpu" if args.dist_backend == "gloo" else None)
    else:
        m = engine.Micro(n_g, W, density=d, initial_threshold=delta0, scaling_factor=ALPHA, dense_output=args.dense,
                         record_error_norm=args.error_norm, sparsifier=args.sparsifier, dtype=tdt)
    stream = torch.cuda.current_stream(dev)
    # the model update x -= g/n at the union is part of the reference's
    # iteration (harness.cpp:212-215); a dense g/n is not (run_iteration uses
    # the sparse sums), so it is materialised only with --dense
    model = torch.zeros(n_g, device=dev, dtype=tdt)
    if args.model:
        m.set_model(model)

    # The threshold adapts for `prime` untimed iterations on fresh N(0,1)
    # gradients (generated between steps), reaching the stationary regime the
    # density target refers to.  The warm-up and timed steps
    # then read gradients that are already resident in HBM: one fresh buffer
    # per step when memory allows (same statistics as the prime phase),
    # otherwise R buffers rotated.
    t = 0
    gen = [torch.empty(n_g, device=dev, dtype=tdt) for _ in range(W)]
    for _ in range(args.prime):
        for i in range(W):
            engine.synth_gaussian(gen[i], args.seed, rank + i, t)
        m.step(gen, ETA, t)
        t += 1
    del gen
    torch.cuda.synchronize()
    need = (args.warmup + args.steps) * W
    R = max(W + 1, min(need, args.buffers, int(0.6 * torch.cuda.mem_get_info(dev)[0] // (esz * n_g))))
    G = [torch.empty(n_g, device=dev, dtype=tdt) for _ in range(R)]
    for r in range(R):
        engine.synth_gaussian(G[r], args.seed, rank + r % W, t + r)
    t0_bufs = t

    def grads(t):
        q = (t - t0_bufs) * W
        return [G[(q + i) % R] for i in range(W)]

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
    # 4th step of the timed region (an event pair between kernels costs the
    # step ~5 µs at c1 size; sampled, the step time stays the step's)
    m.kernel_timing(True, every=4)
    if dist:
        m.exchange_timing(True)
    # the step's working set (e, G, x) fits in L2 at the small workloads:
    # there, flush L2 between timed steps (a 256 MB write, outside the per-step
    # event windows); at C3 and up the inputs are larger than L2
    flush = args.flush_l2 == "on" or (args.flush_l2 == "auto" and 3 * esz * n_g < 2 * 126e6)
    scratch = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if flush else None
    step_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)] if flush else []
    with ClockSampler(local) as clk:
        start.record(stream)
        for s in range(args.steps):
            if flush:
                scratch.fill_(s & 0xFF)
                step_ev[s][0].record(stream)
            m.step(grads(t), ETA, t)  # the whole iteration, one library call
            if flush:
                step_ev[s][1].record(stream)
            t += 1
        end.record(stream)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in step_ev]
    total_ms = sum(step_ms) if flush else start.elapsed_time(end)
    k1a_ms = [float(v) for v in m.kernel_times(args.steps)]  # k1_stream alone (sampled launches)
    m.kernel_timing(False)
    xchg_ms = None
    if dist:
        xt = m.exchange_times()
        m.exchange_timing(False)
        v = torch.tensor([statistics.mean(xt) if xt else 0.0],
                         device=dev if args.dist_backend == "nccl" else "cpu", dtype=torch.float64)
        dist.all_reduce(v, op=dist.ReduceOp.MAX)
        xchg_ms = float(v[0])
    if dist:
        v = torch.tensor([total_ms], device=dev if args.dist_backend == "nccl" else "cpu", dtype=torch.float64)
        dist.all_reduce(v, op=dist.ReduceOp.MAX)
        total_ms = float(v[0])
    ms_step = total_ms / args.steps
    hist = m.history(args.steps)
    K = hist["K"].astype(np.float64)
    k_own = hist["counts"][:, 0].astype(np.float64)
    density = float(K.mean() / n_g)
    # (dense has no selection pass: the whole step stands in for the kernel)
    k1a_avg_ms = statistics.mean(k1a_ms) if k1a_ms else ms_step
    # algorithmic bytes of the dominant kernel, k1_stream: read e and G, write
    # e (all n_g) + one (int32, value) pair per selection
    # (top-k's compaction pass reads acc only, 1 element read per entry: the
    # histogram passes already wrote acc into e; CLT-k's leader is top-k, its
    # other workers select by threshold — the timed launches average over both)
    acc_only = {"topk": W, "cltk": 1}.get(args.sparsifier, 0)
    k1_bytes = (esz * n_g * (acc_only + 3.0 * (W - acc_only)) / W) + (4.0 + esz) * float(k_own.mean())
    achieved = k1_bytes / (k1a_avg_ms * 1e-3) / 1e9
    peak, peak_kind = peaks()
    # whole step vs the same roofline: K1 bytes + union (8 B) and, with the
    # model update, x read+write (8 B) per union entry
    step_bytes = (W * k1_bytes + (4.0 + esz) * float(K.mean()) + (2.0 * esz * float(K.mean()) if args.model else 0.0)
                  + (2.0 * esz * float(K.mean()) * W if W > 1 else 0.0))  # cluster reduce: W reads + zeroing
    # our kernels per step: k1_stream, k1_gather (+ threshold update + model
    # update) at n = 1; a W-worker cluster: 2 per worker + k_cluster_reduce +
    # k_finalize; n > 1 ranks: K1 x2, gather_foreign, owner_reduce,
    # build_union, finalize (NCCL kernels not counted)
    launches_per_step = ((2 if W == 1 else 2 * W + 2) if world == 1
                         else {"peer": 5, "peer_pull": 4, "nccl": 6}[m.transport])  # K1 x2 + exchange + finalize
    if args.sparsifier != "micro":  # baselines.cuh: per selecting worker, top-k = init + 2 per digit +
        # tie count/find + stream + gather (fp32: 11), hard = 2, else accumulate + count = 2; then
        # union marks (W) + popcount + scan (2) + emit + reduce + finalize (dense: iota + reduce + finalize)
        per = {"topk": 11 * W, "cltk": 11 + 2 * (W - 1), "hard": 2 * W, "dense": 2 * W}[args.sparsifier]
        launches_per_step = per + (3 if args.sparsifier == "dense" else W + 6)
    clocks = clk.summary()

    # ---- end to end through the public API with host buffers (N = 1) ----
    e2e = None
    if world == 1:
        # one distinct pinned host gradient per e2e step (the same statistics
        # as the timed steps; re-feeding one gradient would make the residual
        # grow coherently and inflate the selection)
        ke = max(3, min(args.steps, 10))
        nb = int(max(2, min(ke + 1, 8e9 // (esz * n_g * W))))  # <= 8 GB of pinned host gradients
        hGs = []
        for b in range(nb):
            hG = torch.empty(W * n_g, dtype=tdt).pin_memory()
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
        for s in range(ke):
            i_, _s = m.step_host(hGs[s % (nb - 1)], ETA, t, idx, sums)
            kk.append(i_.size)
            t += 1
        e2e_s = (time.perf_counter() - t0) / ke
        e2e = {"value": e2e_s * 1e6, "unit": "us/iter", "h2d_bytes_per_step": esz * n_g * W,
               "d2h_bytes_per_step": int((4 + esz) * statistics.mean(kk) + 8 + 4),
               "host_gradients": f"{nb - 1} distinct pinned buffers over {ke} steps",
               "density": float(statistics.mean(kk)) / n_g,
               # what bounds it: the H2D of the gradient over PCIe (Gen5 x16: ~64 GB/s nominal)
               "h2d_gbs_effective": esz * n_g * W / e2e_s / 1e9}
    else:
        # N ranks: each copies its own pinned host gradient in, steps through
        # DistMicro, and reads the union back; the max over ranks is reported
        ke = max(3, min(args.steps, 10))
        nb = int(max(2, min(ke + 1, 4e9 // (esz * n_g))))
        hGs = []
        for b in range(nb):
            engine.synth_gaussian(G[0], args.seed, rank, t + 1 + b)
            hGs.append(G[0].cpu().pin_memory())
        dG = torch.empty(n_g, device=dev, dtype=tdt)
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
        v = torch.tensor([(time.perf_counter() - t0) / ke], device=dev if args.dist_backend == "nccl" else "cpu",
                         dtype=torch.float64)
        dist.all_reduce(v, op=dist.ReduceOp.MAX)
        e2e = {"value": float(v[0]) * 1e6, "unit": "us/iter", "h2d_bytes_per_step": esz * n_g,
               "d2h_bytes_per_step": int((4 + esz) * statistics.mean(kk) + 8 + 4),
               "host_gradients": f"{nb - 1} distinct pinned buffers per rank over {ke} steps",
               "density": float(statistics.mean(kk)) / n_g, "per": "rank (max over ranks)"}

    # ---- CPU baseline: the reference's own code on this host (rank 0, N = 1) ----
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            times = run_reference_cluster(n_g, W, d, steps=args.cpu_steps, warmup=1)
            cpu = {"value": statistics.mean(times) * 1e6, "unit": "us/iter", "cores": 1, "kind": "reference",
                   "sample": f"{args.cpu_steps} iterations (after 1 warm-up) of the full workload (n_g={n_g}, n={W}) "
                             "through the reference's sparsifier/collectives TUs compiled verbatim (fp64, 1 thread)"}
        except Exception as ex:  # the checker is optional at run time; the GPU number stands
            cpu = {"value": None, "unit": "us/iter", "cores": 1, "kind": "reference", "sample": f"failed: {ex}"}

    # the exchange against the NVLink roofline (N > 1): bytes received per GPU,
    # 4(K-k) foreign indices + 4k(n-1) contributions + 4(K-k) sums
    exchange_line = None
    if dist and xchg_ms:
        Km, km = float(K.mean()), float(k_own.mean())
        b_net = 4.0 * (Km - km) + 4.0 * km * (world - 1) + 4.0 * (Km - km)
        exchange_line = {"bound": "nvlink", "achieved": b_net / (xchg_ms * 1e-3) / 1e9, "peak": 900.0,
                         "unit": "GB/s", "frac": b_net / (xchg_ms * 1e-3) / 1e9 / 900.0,
                         "bytes_per_gpu": b_net, "avg_ms": xchg_ms, "transport": m.transport,
                         "peak_source": "NVLink 5 per direction per GPU (nominal)",
                         "timed": "exchange kernels, barriers excluded" if m.transport != "nccl"
                         else "the whole NCCL protocol"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": ms_step * 1e3, "unit": "us/iter", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": False, "scaling": "weak",
            "vs_baseline": None, "dtype": args.dtype,
            "data": f"synthetic N(0,1) {args.dtype} gradients (include/micro_synth.h)",
            "config": {"workload": wl["desc"], "n_g": n_g, "density_target": d, "workers": world * W,
                       "one_worker_per_gpu": W == 1, "eta": ETA, "alpha": ALPHA, "delta0": delta0,
                       "adaptation_iterations": args.prime, "first_timed_t": t_first,
                       "model_update": bool(args.model), "dense_g_over_n": bool(args.dense),
                       "error_norm_recorded": bool(args.error_norm), "seed": args.seed,
                       "sparsifier": args.sparsifier,
                       "inputs": (f"{R} resident N(0,1) gradients ("
                                  + ("one fresh per step" if R >= args.warmup + args.steps else "rotated")
                                  + (f"); L2 flushed between timed steps (256 MB write outside the per-step "
                                     f"events: the working set {3 * esz * n_g / 1e6:.0f} MB would fit L2)"
                                     if flush else f"); each {esz}*n_g bytes > L2 (no flush needed)"
                                     if esz * n_g > 126e6 else "); L2 NOT flushed (--flush-l2 off)")),
                       "parallelism": (f"dp{world} (exclusive cyclic partitions"
                                       + (f", {m.transport} exchange)" if world > 1 else ")") if W == 1 else
                                       f"{W} in-process workers on 1 GPU (exclusive cyclic partitions)")},
            "median_us_per_step": (float(np.median(step_ms)) * 1e3 if step_ms else None),
            "density": density, "density_rel_err": density / d - 1.0,
            "density_window": {"first_quarter": float(K[: max(1, len(K) // 4)].mean() / n_g),
                               "last_quarter": float(K[-max(1, len(K) // 4):].mean() / n_g),
                               "median": float(np.median(K) / n_g)},
            "select_gbs": achieved,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic_from_profiles(args.workload),
                         "kernel": "k1_stream", "algorithmic_bytes_per_launch": k1_bytes,
                         "avg_launch_ms": k1a_avg_ms, "peak_source": peak_kind,
                         "timed_launches": f"{len(k1a_ms)} of {args.steps} (every 4th, CUDA events on the launch stream)",
                         "step_frac": step_bytes / (ms_step * 1e-3) / 1e9 / peak},
            "exchange": exchange_line,
            "clocks": clocks,
            "gpu_launches": launches_per_step * args.steps,
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="c3")
    ap.add_argument("--prime", type=int, default=1000, help="untimed threshold-adaptation iterations")
    ap.add_argument("--buffers", type=int, default=256, help="max resident gradient buffers")
    ap.add_argument("--cpu-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dense", action="store_true", help="also maintain the dense g/n vector")
    ap.add_argument("--cluster-workers", type=int, default=1,
                    help="N = 1 only: W in-process workers on the GPU (the reference's in-process cluster)")
    ap.add_argument("--no-model", dest="model", action="store_false", help="skip the model update x -= g/n")
    ap.add_argument("--sparsifier", choices=["micro", "topk", "cltk", "hard", "dense"], default="micro",
                    help="N = 1: a comparison sparsifier of the reference's harness instead of MiCRO")
    ap.add_argument("--dist-backend", choices=["nccl", "gloo"], default="nccl",
                    help="gloo: exercise the N > 1 path with all ranks on one GPU (code check only)")
    ap.add_argument("--transport", choices=["peer", "peer_pull", "nccl"], default="peer",
                    help="N > 1: exchange over peer memory (one kernel per rank) or the NCCL protocol")
    ap.add_argument("--seed", type=int, default=SEED, help="synthetic gradient stream (SURVEY.md 8d: 1, 2, 3)")
    ap.add_argument("--flush-l2", choices=["auto", "on", "off"], default="auto",
                    help="flush L2 between timed steps (auto: when e, G and x would fit in L2)")
    ap.add_argument("--dtype", choices=["f32", "f64"], default="f32",
                    help="f64: the reference's own arithmetic (bit-exact with its code)")
    ap.add_argument("--error-norm", action="store_true",
                    help="also record the per-step error norm ||e_{t+1}|| (fused into k1_stream); off by "
                         "default, like the reference arm's timed step")
    args = ap.parse_args()
    wl = WORKLOADS[args.workload]
    if args.impl == "reference":
        return reference_arm(args, wl)
    return our_arm(args, wl)


if __name__ == "__main__":
    sys.exit(main())
