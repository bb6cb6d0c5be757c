"""bench.py --impl reference (the reference's own code on the host CPU, no
GPU): the JSON line's contract and the stationary-regime protocol."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_line():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--workload", "c1", "--steps", "2",
                        "--warmup", "1", "--prime", "1600"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert d["impl"] == "reference" and d["dtype"] == "f64" and d["higher_is_better"] is False
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] == d["host"]["threads_used"] == 1
    assert d["config"]["n_g"] == 11_700_000 and d["config"]["dense_g_over_n"] and d["config"]["model_update"]
    assert d["protocol"]["first_timed_t"] == 1601
    assert d["config"]["alpha"] == 0.001
    # past the controller's adaptation (alpha = 0.001: ~1300 iterations from
    # the warm start): within 10 % of d = 1 % (stationary ~1.00 %)
    assert 0.009 < d["density"] < 0.011, d["density"]
