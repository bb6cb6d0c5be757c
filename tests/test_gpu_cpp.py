"""The C++ hosts of the C ABI: the drop-in (include/sparsim_b200.hpp)
passes the reference's hot-path unit tests, restated in
tests/cpp/test_dropin.cpp; and an n-rank step driven from C++ alone, one
process per rank over CUDA IPC (tests/cpp/test_dist_ipc.cpp).  GPU only."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu


def test_cpp_dropin_suite():
    from paper_2310_00967_b200.build import CPP_TEST_BIN, build_cpp_tests, cpp_tests_stale
    if cpp_tests_stale():
        build_cpp_tests()
    r = subprocess.run([CPP_TEST_BIN], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "OK: 0 failed checks" in r.stdout


def test_cpp_n_process_peer_exchange():
    from paper_2310_00967_b200.build import CPP_BIN_DIR, build_cpp_tests, cpp_tests_stale
    exe = os.path.join(CPP_BIN_DIR, "test_dist_ipc")
    if cpp_tests_stale():
        build_cpp_tests()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "world 2:" in r.stdout and "world 3:" in r.stdout and "OK: 0 failing cases" in r.stdout
