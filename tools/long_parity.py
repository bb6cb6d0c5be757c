"""Long at-size parity runs (evidence beyond the pytest budget): the CUDA path
and the checker stepped together every iteration, as tests/test_gpu_configs.py
does, for longer than the suite can afford.

    python tools/long_parity.py [out.json] [--more]

  c3_n1_f64_g32: the bench's default step (138M, d = 0.01, n = 1, fp32
      gradients into fp64 state, model + dense g/n) vs the reference's own
      compiled code (oracle/_ref), 150 iterations from the warm delta_0.
  c3_n8_f32: 138M, n = 8, the in-process cluster and the 8-rank peer
      exchange (GroupMicro) vs the C restatement, 20 iterations.
  --more: C1 (n = 1, fp32) for 2000 iterations (the reference's acceptance-run
      length, acceptance.cpp:93-118), C4 for 30, C5 d = 0.1 / 0.001 for 10.
  --baselines: top-k / CLT-k / hard threshold at C1 x 8, 20 iterations.
  --ref: C1 fp64 on fp32 gradients vs the reference's own code for 2000
      iterations; C2 at n = 8 (cluster + GroupMicro) for 200.
Every iteration: counts, union indices and sums, next thresholds (exact);
residuals, model and dense g/n at the listed checkpoints."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for _p in (ROOT, os.path.join(ROOT, "oracle")):  # as tests/conftest.py
    sys.path.insert(0, _p)
from tests.test_gpu_configs import Run, warm_delta0  # noqa: E402


OUT = "gpurun_out/long_parity.json"
RES = []


def long_run(tag, iters, checks, **kw):
    t0 = time.time()
    run = Run(**kw)
    for t in range(iters):
        run.step(t, full_check=t in checks)
    run.close()
    r = {"case": tag, "iterations": iters, "full_checks_at": sorted(checks), "result": "bit-exact",
         "wall_s": round(time.time() - t0, 1)}
    RES.append(r)
    with open(OUT, "w") as f:  # after every case: a later failure keeps the earlier results
        json.dump(RES, f, indent=1)
    return r


def more(res):
    """The acceptance-run length at C1 and longer runs at C4 / C5."""
    res.append(long_run("c1_n1_f32 vs restatement (acceptance length)", 2000, {0, 999, 1999}, n_g=11_700_000, n=1,
                        d=0.01, delta0=0.01))
    print(json.dumps(res[-1]), flush=True)
    res.append(long_run("c4_n1_f32 vs restatement", 30, {29}, n_g=340_000_000, n=1, d=0.001,
                        delta0=warm_delta0(0.001)))
    print(json.dumps(res[-1]), flush=True)
    for d in (0.1, 0.001):
        res.append(long_run(f"c5_n1_d{d}_f32 vs restatement", 10, {9}, n_g=1_500_000_000, n=1, d=d,
                            delta0=warm_delta0(d)))
        print(json.dumps(res[-1]), flush=True)


def ref_long(res):
    """The acceptance-run length against the reference's own code (fp64), and
    the partitioned C2 cluster + peer exchange over 200 iterations."""
    res.append(long_run("c1_n1_f64_g32 vs reference code (acceptance length)", 2000, {0, 999, 1999},
                        n_g=11_700_000, n=1, d=0.01, delta0=0.01, dtype=np.float64, checker="reference",
                        grad32=True))
    print(json.dumps(res[-1]), flush=True)
    res.append(long_run("c2_n8_f32 cluster + GroupMicro vs restatement", 200, {0, 99, 199}, n_g=11_700_000, n=8,
                        d=0.01, delta0=warm_delta0(0.01), group=True))
    print(json.dumps(res[-1]), flush=True)


def baselines(res):
    """The comparison sparsifiers at C1 x 8 (batched top-k, union by words /
    by gather) vs the restatement (BaselineCluster), 20 iterations, every
    quantity every iteration (tests/test_gpu_baselines.py's run)."""
    from tests.test_gpu_baselines import run as brun
    kinds = os.environ.get("KINDS", "topk,cltk,hard").split(",")
    for kind, delta0 in (("topk", 0.02), ("cltk", 0.02), ("hard", 0.0258)):
        if kind not in kinds:
            continue
        t0 = time.time()
        Ks = brun(kind, 11_700_000, 8, 0.01, False, iters=20, delta0=delta0)
        r = {"case": f"c1_n8_{kind}_f32 vs restatement", "iterations": 20, "full_checks_at": list(range(20)),
             "result": "bit-exact", "union_density": [round(K / 11_700_000, 4) for K in Ks[:3]] + ["..."] +
             [round(Ks[-1] / 11_700_000, 4)], "wall_s": round(time.time() - t0, 1)}
        RES.append(r)
        with open(OUT, "w") as f:
            json.dump(RES, f, indent=1)
        res.append(r)
        print(json.dumps(r), flush=True)


def main():
    global OUT
    OUT = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("--") else OUT
    res = []
    if "--baselines" in sys.argv:
        baselines(res)
        return
    if "--ref" in sys.argv:
        ref_long(res)
        return
    if "--more" in sys.argv:
        more(res)
        return
    res.append(long_run("c3_n1_f64_g32 vs reference code", 150, {0, 49, 99, 149}, n_g=138_000_000, n=1, d=0.01,
                        delta0=warm_delta0(0.01), dtype=np.float64, checker="reference", grad32=True))
    print(json.dumps(res[-1]), flush=True)
    res.append(long_run("c3_n8_f32 cluster + GroupMicro vs restatement", 20, {0, 9, 19}, n_g=138_000_000, n=8,
                        d=0.01, delta0=warm_delta0(0.01), group=True))
    print(json.dumps(res[-1]), flush=True)


if __name__ == "__main__":
    main()
