"""bench.py's contract on the GPU: the JSON line's keys at N = 1, and the
N = 2 path (both ranks on one GPU over gloo: a code-path check, the numbers
are not valid) for each exchange transport.  GPU only."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "clocks", "gpu_launches"}


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _line(out: str) -> dict:
    return json.loads([ln for ln in out.splitlines() if ln.startswith("{")][-1])


def test_bench_line_n1():
    r = subprocess.run([sys.executable, "bench.py", "--workload", "c1", "--steps", "5", "--warmup", "3", "--prime",
                        "50", "--cpu-steps", "1"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _line(r.stdout)
    assert KEYS <= set(d), KEYS - set(d)
    assert d["n_gpus"] == 1 and d["higher_is_better"] is False and d["gpu_launches"] == 2 * 5
    assert set(d["roofline"]) >= {"bound", "achieved", "peak", "unit", "frac", "traffic"}
    assert set(d["e2e"]) >= {"value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"}
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] == 1
    assert d["dtype"] == "f64" and d["config"]["dense_g_over_n"] and d["config"]["model_update"]
    assert d["other_dtype"]["dtype"] == "f32" and d["other_dtype"]["value"] > 0
    # the reference arm runs the identical workload
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--workload", "c1", "--steps", "2",
                        "--warmup", "1", "--prime", "50"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    ref = _line(r.stdout)
    assert ref["impl"] == "reference" and ref["config"] == d["config"] and ref["metric"] == d["metric"]


@pytest.mark.parametrize("transport", ["peer", "peer_pull", "nccl"])
def test_bench_n2_code_path(transport):
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py",
                        "--gpus", "2", "--dist-backend", "gloo", "--transport", transport, "--workload", "c1",
                        "--steps", "3", "--warmup", "3", "--prime", "20"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _line(r.stdout)
    assert d["n_gpus"] == 2 and d["e2e"]["per"].startswith("rank")
    assert d["exchange"]["bound"] == "nvlink" and d["exchange"]["avg_ms"] > 0
    assert transport in d["config"]["parallelism"]
