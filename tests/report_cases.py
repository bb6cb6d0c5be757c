"""Record sets for the report-format tests (shared by tests/test_report.py
and tests/golden/make_report_golden.py)."""
import numpy as np

from paper_2310_00967_b200.report import RunConfig


def _records(n, seed, zero_norm=False):
    rng = np.random.default_rng(seed)
    out = []
    for t in range(n):
        out.append({"t": t, "actual_density": float(rng.uniform(0.005, 0.02)),
                    "buildup_factor": float(rng.uniform(0.9, 1.3)), "redundant_traffic_factor": 1.0,
                    "error_norm": 0.0 if zero_norm else float(rng.standard_normal() ** 2 * 1e-3),
                    "threshold": float(abs(rng.standard_normal()) * 0.03), "loss": 0.0,
                    "time_grad": 0.0, "time_select": 0.0, "time_comm": 0.0, "time_overhead": 0.0})
    return out


CASES = {
    "micro_default": (RunConfig(), _records(12, 1)),
    "micro_c3": (RunConfig(workers=8, iterations=1000, density=0.01, delta0=0.025758293035489, lr=0.01,
                           per_worker_k="full", error_feedback=False, seed=7),
                 _records(5, 2)),
    "odd_values": (RunConfig(workers=1, density=1.0, delta0=0.0, alpha=0.5, eps_delta=1e-300, lr=3e-7,
                             decay_at=150, bandwidth=1e12, latency_per_collective=1.0 / 3.0, task="mlp2"),
                   [{"t": 0, "actual_density": 1.0, "buildup_factor": 100.0, "redundant_traffic_factor": 0.0,
                     "error_norm": 1e-320, "threshold": 12345678901234.5, "loss": -0.0, "time_grad": 5e-324,
                     "time_select": 1.7976931348623157e308, "time_comm": 0.1, "time_overhead": 2.0 / 3.0}]),
    "zero_norm": (RunConfig(), _records(3, 3, zero_norm=True)),
    "empty": (RunConfig(), []),
}
