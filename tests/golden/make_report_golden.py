"""Golden record files written by the REFERENCE's own report.cpp
(oracle/_ref/libsparsim_report.so, compiled verbatim), so tests/test_report.py
can check report.py byte for byte where /root/reference is absent.

    python tests/golden/make_report_golden.py
"""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]

from oracle import ReferenceReport  # noqa: E402
from tests.report_cases import CASES  # noqa: E402

rep = ReferenceReport()
for name, (cfg, records) in CASES.items():
    for fmt in ("csv", "json"):
        rep.emit(fmt, os.path.join(HERE, f"report_{name}.{fmt}"), records, cfg.to_json())
print("wrote", len(CASES) * 2, "files")
