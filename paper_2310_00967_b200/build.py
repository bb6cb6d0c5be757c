"""Build recipe for the in-tree CUDA library (sm_100a only).

    python -m paper_2310_00967_b200.build          # -> paper_2310_00967_b200/lib/libmicro_b200.so

No fast-math, no FTZ, explicit __f*_rn arithmetic in the kernels: the
accumulate and reduce must round exactly like the reference.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIBDIR, "libmicro_b200.so")
SOURCES = ["api.cu", "dist_api.cu", "value_api.cu", "nccl_api.cu"]
HEADERS = ["internal.cuh", "baselines.cuh", "common.cuh", "norm.cuh", "scan.cuh", "select_stream.cuh",
           "exchange.cuh", "peer.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3",
         "-fmad=false", "-prec-div=true", "-prec-sqrt=true", "-ftz=false",
         "-I", os.path.join(ROOT, "include")]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps += [os.path.join(ROOT, "include", f) for f in ("micro.h", "micro_synth.h")]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    os.makedirs(LIBDIR, exist_ok=True)
    objdir = os.path.join(ROOT, "build", "obj")
    os.makedirs(objdir, exist_ok=True)
    # one nvcc per translation unit, in parallel, then one shared-library link
    objs, procs = [], []
    for src in SOURCES:
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        objs.append(obj)
        procs.append(subprocess.Popen([NVCC, *ARCH, *FLAGS, *(["-Xptxas", "-v"] if verbose else []),
                                       "-c", "-o", obj, os.path.join(CSRC, src)]))
    if any(p.wait() != 0 for p in procs):
        raise subprocess.CalledProcessError(1, "nvcc")
    subprocess.run([NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-ldl"], check=True)
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose="-v" in sys.argv))


CPP_TESTS = {  # name -> source: the C++ hosts of the C ABI (no Python on their path)
    "test_dropin": os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp"),
    "test_dist_ipc": os.path.join(ROOT, "tests", "cpp", "test_dist_ipc.cpp"),
}
CPP_BIN_DIR = os.path.join(ROOT, "tests", "cpp", "build")
CPP_TEST_BIN = os.path.join(CPP_BIN_DIR, "test_dropin")


def cpp_tests_stale() -> bool:
    """A C++ test binary older than its source, the headers or the library
    (a micro_config layout change must never meet an old binary)."""
    deps = [os.path.join(ROOT, "include", f) for f in ("micro.h", "sparsim_b200.hpp", "micro_synth.h")] + [LIB]
    for name, src in CPP_TESTS.items():
        exe = os.path.join(CPP_BIN_DIR, name)
        if not os.path.exists(exe):
            return True
        t = os.path.getmtime(exe)
        if any(os.path.getmtime(d) > t for d in deps + [src] if os.path.exists(d)):
            return True
    return False


def build_cpp_tests() -> str:
    """The reference's hot-path unit tests restated against the C++ drop-in
    header (include/sparsim_b200.hpp), and the n-process C++ host of the
    peer exchange, linked against the in-tree library."""
    build()
    os.makedirs(CPP_BIN_DIR, exist_ok=True)
    for name, src in CPP_TESTS.items():
        subprocess.run(["g++", "-std=c++20", "-O2", "-Wall", "-I", os.path.join(ROOT, "include"), src,
                        "-L", LIBDIR, "-lmicro_b200", "-pthread",
                        "-Wl,-rpath,$ORIGIN/../../../paper_2310_00967_b200/lib",
                        "-o", os.path.join(CPP_BIN_DIR, name)], check=True)
    return CPP_TEST_BIN
