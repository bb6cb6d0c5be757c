"""Reference-format records (report.py) — byte for byte the reference's own
report.cpp (compiled verbatim in oracle/_ref): live where the reference is
built, and against the committed golden files it wrote
(tests/golden/make_report_golden.py) everywhere.  CPU only."""
import os

import pytest

from paper_2310_00967_b200 import report
from tests.report_cases import CASES

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.mark.parametrize("name", sorted(CASES))
@pytest.mark.parametrize("fmt", ["csv", "json"])
def test_matches_reference_golden(name, fmt, tmp_path):
    cfg, recs = CASES[name]
    out = tmp_path / f"r.{fmt}"
    report.emit(cfg, recs, fmt, str(out))
    with open(os.path.join(GOLDEN, f"report_{name}.{fmt}"), "rb") as f:
        want = f.read()
    assert out.read_bytes() == want


@pytest.mark.ref
@pytest.mark.parametrize("fmt", ["csv", "json"])
def test_matches_reference_live(fmt, tmp_path):
    from oracle import ReferenceReport
    ref = ReferenceReport()
    for name, (cfg, recs) in CASES.items():
        a, b = tmp_path / f"a_{name}.{fmt}", tmp_path / f"b_{name}.{fmt}"
        report.emit(cfg, recs, fmt, str(a))
        ref.emit(fmt, str(b), recs, cfg.to_json())
        assert a.read_bytes() == b.read_bytes(), name


def test_read_back_and_scaling(tmp_path):
    cfg, recs = CASES["micro_default"]
    p = tmp_path / "r.json"
    report.emit(cfg, recs, "json", str(p))
    back = report.read_records_json(str(p))
    assert back["config"] == cfg.to_json()
    assert [r["t"] for r in back["records"]] == [r["t"] for r in recs]
    assert all(a["error_norm"] == b["error_norm"] for a, b in zip(back["records"], recs))
    # metrics.cpp:12-23
    assert report.threshold_error_scaling([1.0, 2.0], [0.5, 0.5]) == 3.0
    assert report.threshold_error_scaling([1.0], [0.0]) is None
    with pytest.raises(ValueError):
        report.threshold_error_scaling([], [])
    with pytest.raises(ValueError):
        report.emit(cfg, recs, "xml", str(p))
