"""The C++ drop-in (include/sparsim_b200.hpp) passes the reference's
hot-path unit tests, restated in tests/cpp/test_dropin.cpp.  GPU only."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu


def test_cpp_dropin_suite():
    from paper_2310_00967_b200.build import CPP_TEST_BIN, build_cpp_tests
    if not os.path.exists(CPP_TEST_BIN):
        build_cpp_tests()
    r = subprocess.run([CPP_TEST_BIN], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "OK: 0 failed checks" in r.stdout
