"""Long at-size parity runs (evidence beyond the pytest budget): the CUDA path
and the checker stepped together every iteration, as tests/test_gpu_configs.py
does, for longer than the suite can afford.

    python tools/long_parity.py [out.json]

  c3_n1_f64_g32: the bench's default step (138M, d = 0.01, n = 1, fp32
      gradients into fp64 state, model + dense g/n) vs the reference's own
      compiled code (oracle/_ref), 150 iterations from the warm delta_0.
  c3_n8_f32: 138M, n = 8, the in-process cluster and the 8-rank peer
      exchange (GroupMicro) vs the C restatement, 20 iterations.
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


def long_run(tag, iters, checks, **kw):
    t0 = time.time()
    run = Run(**kw)
    for t in range(iters):
        run.step(t, full_check=t in checks)
    run.close()
    return {"case": tag, "iterations": iters, "full_checks_at": sorted(checks), "result": "bit-exact",
            "wall_s": round(time.time() - t0, 1)}


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/long_parity.json"
    res = []
    res.append(long_run("c3_n1_f64_g32 vs reference code", 150, {0, 49, 99, 149}, n_g=138_000_000, n=1, d=0.01,
                        delta0=warm_delta0(0.01), dtype=np.float64, checker="reference", grad32=True))
    print(json.dumps(res[-1]), flush=True)
    res.append(long_run("c3_n8_f32 cluster + GroupMicro vs restatement", 20, {0, 9, 19}, n_g=138_000_000, n=8,
                        d=0.01, delta0=warm_delta0(0.01), group=True))
    print(json.dumps(res[-1]), flush=True)
    with open(out, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
