"""Reference-format run records: the CSV / JSON files the
reference's `sparsim::emit` writes (report.hpp:1-46, report.cpp:11-119), from
the records of a GPU run (`Micro.records()` / `DistMicro.records()`), so the
reference's plotting and acceptance tooling reads GPU output unchanged.

Byte-for-byte the reference's layout (checked against its own report.cpp,
compiled verbatim in oracle/_ref, by tests/test_report.py):

* CSV: ``# key=value`` lines of the run configuration (keys sorted, as
  nlohmann's std::map orders them; strings bare, everything else JSON),
  ``# threshold_error_scaling=<%.17g|none>``, the column row, then one row
  per iteration with every double printed ``%.17g``.
* JSON: ``{"config", "error_norm_scaled", "records",
  "threshold_error_scaling"}`` (sorted keys, indent 2).

The MiCRO path fills t, actual_density, buildup_factor,
redundant_traffic_factor, error_norm and threshold; loss and the modeled
phase times belong to the simulator's task and cost model (out of scope) and
are 0 unless the caller supplies them.
"""
from __future__ import annotations

import json
import math
from dataclasses import dataclass, field
from typing import Iterable, Sequence

COLUMNS = ("iter,actual_density,buildup_factor,redundant_traffic_factor,error_norm,"
           "error_norm_scaled,threshold,loss,time_grad,time_select,time_comm,time_overhead")
RECORD_FIELDS = ("actual_density", "buildup_factor", "redundant_traffic_factor", "error_norm", "threshold",
                 "loss", "time_grad", "time_select", "time_comm", "time_overhead")
TASKS = ("quadratic", "logreg", "mlp2")                      # task.cpp:348-355
SPARSIFIERS = ("micro", "topk", "cltk", "hard", "dense")     # sparsifier.cpp:127-135


@dataclass
class RunConfig:
    """harness.hpp:34-47 with the reference's defaults (LrSchedule
    harness.hpp:24-31, SparsifierConfig sparsifier.hpp:39-46,
    CostModelParams collectives.hpp:46-50)."""
    workers: int = 4
    iterations: int = 200
    batch_size: int = 8
    seed: int = 42
    task: str = "quadratic"
    dimension: int = 0
    samples: int = 0
    sparsifier: str = "micro"
    density: float = 0.01
    delta0: float = 0.01
    alpha: float = 0.01
    eps_delta: float = 1e-12
    per_worker_k: str = "split"
    lr: float = 0.01
    decay_factor: float = 0.1
    decay_at: int = -1
    error_feedback: bool = True
    latency_per_collective: float = 25e-6
    bytes_per_element: float = 8.0
    bandwidth: float = 1.25e9
    compute_time_per_op: float = 1e-9
    extra: dict = field(default_factory=dict)  # not written (the reference has no such keys)

    def to_json(self) -> dict:
        """config_to_json (report.cpp:97-119)."""
        if self.task not in TASKS or self.sparsifier not in SPARSIFIERS or self.per_worker_k not in ("split", "full"):
            raise ValueError("config: unknown task / sparsifier / per_worker_k name")
        return {"sparsifier": self.sparsifier, "task": self.task, "workers": int(self.workers),
                "iterations": int(self.iterations), "batch_size": int(self.batch_size), "seed": int(self.seed),
                "dimension": int(self.dimension), "samples": int(self.samples), "density": float(self.density),
                "delta0": float(self.delta0), "alpha": float(self.alpha), "eps_delta": float(self.eps_delta),
                "per_worker_k": self.per_worker_k, "lr": float(self.lr), "decay_factor": float(self.decay_factor),
                "decay_at": int(self.decay_at), "error_feedback": bool(self.error_feedback),
                "latency_per_collective": float(self.latency_per_collective),
                "bytes_per_element": float(self.bytes_per_element), "bandwidth": float(self.bandwidth),
                "compute_time_per_op": float(self.compute_time_per_op)}


def _g17(v: float) -> str:
    return "%.17g" % v


def _jnum(v):
    """A JSON value as nlohmann prints it (NaN/inf become null)."""
    if isinstance(v, float) and not math.isfinite(v):
        return None
    return v


def threshold_error_scaling(deltas: Sequence[float], errors: Sequence[float]) -> float | None:
    """metrics.cpp:12-23: sum(deltas) / sum(errors), None when the error sum is 0."""
    if len(deltas) == 0 or len(deltas) != len(errors):
        raise ValueError("threshold_error_scaling: series must be nonempty and equal length")
    ds = es = 0.0
    for d in deltas:
        ds += float(d)
    for e in errors:
        es += float(e)
    if es == 0.0:
        return None
    return ds / es


def _rows(records: Iterable[dict]) -> list[dict]:
    out = []
    for r in records:
        row = {"t": int(r["t"])}
        for f in RECORD_FIELDS:
            row[f] = float(r.get(f, 0.0))
        out.append(row)
    return out


def _scaling(rows) -> float | None:
    if not rows:
        return None
    return threshold_error_scaling([r["threshold"] for r in rows], [r["error_norm"] for r in rows])


def to_csv(config: RunConfig, records: Iterable[dict]) -> str:
    """emit_csv (report.cpp:33-55)."""
    rows = _rows(records)
    sc = _scaling(rows)
    lines = []
    for k, v in sorted(config.to_json().items()):
        lines.append(f"# {k}=" + (v if isinstance(v, str) else json.dumps(v)))
    lines.append("# threshold_error_scaling=" + (_g17(sc) if sc is not None else "none"))
    lines.append(COLUMNS)
    factor = sc if sc is not None else 0.0
    for r in rows:
        vals = [r["actual_density"], r["buildup_factor"], r["redundant_traffic_factor"], r["error_norm"],
                r["error_norm"] * factor, r["threshold"], r["loss"], r["time_grad"], r["time_select"],
                r["time_comm"], r["time_overhead"]]
        lines.append(str(r["t"]) + "," + ",".join(_g17(v) for v in vals))
    return "\n".join(lines) + "\n"


def to_json(config: RunConfig, records: Iterable[dict]) -> str:
    """emit_json (report.cpp:57-83): nlohmann::json dump(2), keys sorted."""
    rows = _rows(records)
    sc = _scaling(rows)
    factor = sc if sc is not None else 0.0
    doc = {"config": config.to_json(), "threshold_error_scaling": _jnum(sc),
           "error_norm_scaled": [_jnum(r["error_norm"] * factor) for r in rows],
           "records": [{k: _jnum(v) for k, v in r.items()} for r in rows]}
    return json.dumps(doc, indent=2, sort_keys=True, allow_nan=False) + "\n"


def emit(config: RunConfig, records: Iterable[dict], fmt: str, path: str) -> None:
    """sparsim::emit (report.cpp:121-131)."""
    if fmt not in ("csv", "json"):
        raise ValueError(f"unknown format '{fmt}' (expected csv|json)")
    text = to_csv(config, records) if fmt == "csv" else to_json(config, records)
    with open(path, "w", newline="") as f:
        f.write(text)


def read_records_json(path: str) -> dict:
    """read_records_json (report.hpp:38-44): config, threshold_error_scaling, records."""
    with open(path) as f:
        j = json.load(f)
    recs = []
    for r in j["records"]:
        d = {"t": int(r["t"])}
        for k in RECORD_FIELDS:
            v = r.get(k)
            d[k] = float("nan") if v is None else float(v)
        recs.append(d)
    return {"config": j["config"], "threshold_error_scaling": j.get("threshold_error_scaling"), "records": recs}


def config_for(m, lr: float, iterations: int, **kw) -> RunConfig:
    """The RunConfig of a run driven through engine.Micro / dist.DistMicro."""
    c = m.cfg if hasattr(m, "cfg") else m.m.cfg
    return RunConfig(workers=c.n_workers, iterations=iterations, density=c.density, delta0=c.initial_threshold,
                     alpha=c.scaling_factor, eps_delta=c.min_threshold,
                     per_worker_k="split" if c.target == 0 else "full", lr=lr,
                     error_feedback=bool(c.error_feedback), **kw)
