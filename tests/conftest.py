import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "ref: needs oracle/_ref (the reference's own code, built where /root/reference exists)")


def _ref_available():
    return os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libsparsim_ref.so")) or os.path.isdir(
        "/root/reference/proj/src")


def pytest_collection_modifyitems(config, items):
    if _ref_available():
        return
    skip = pytest.mark.skip(reason="oracle/_ref not built and /root/reference absent")
    for it in items:
        if "ref" in it.keywords:
            it.add_marker(skip)
