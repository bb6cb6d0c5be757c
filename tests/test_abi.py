"""The C-ABI library loads, exports every symbol include/micro.h declares, and
its pure host functions reproduce the reference KATs.  CPU only: no device
work is attempted except to check that it fails loudly without a GPU."""
import ctypes as C
import os
import re

import numpy as np
import pytest
import torch

from oracle import Oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_2310_00967_b200 import _lib
    return _lib.lib()


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "micro.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(micro_[a-z0-9_]+)\s*\(", src)))


def test_every_declared_symbol_is_exported(L):
    from paper_2310_00967_b200 import _lib
    syms = declared_symbols()
    assert len(syms) >= 35
    for s in syms:
        assert hasattr(L, s), s
    assert sorted(_lib.EXPORTED) == syms


def test_host_partition_and_targets_match_oracle(L):
    from paper_2310_00967_b200 import sparsim
    o = Oracle()
    rng = np.random.default_rng(3)
    for _ in range(300):
        n = int(rng.integers(1, 17))
        n_g = n + int(rng.integers(0, 100_000))
        t = int(rng.integers(0, 10_000))
        for i in range(n):
            r = sparsim.partition(n_g, n, t, i)
            assert (r.start, r.end) == o.partition(n_g, n, t, i) and r.owner == i
    assert (sparsim.partition(10, 4, 1, 3).start, sparsim.partition(10, 4, 1, 3).end) == (0, 3)
    with pytest.raises(ValueError, match="smaller than worker count"):
        sparsim.partition(3, 4, 0, 0)
    assert sparsim.global_target_count(0.01, 10000) == 100
    assert sparsim.per_worker_target_count(0.001, 10000, 16, "split") == 1
    assert sparsim.per_worker_target_count(0.01, 10000, 4, "full") == 100
    with pytest.raises(ValueError):
        sparsim.global_target_count(1.5, 100)


def test_host_threshold_update(L):
    from paper_2310_00967_b200 import sparsim
    o = Oracle()
    S = sparsim.ThresholdState
    assert sparsim.micro_update_threshold(S(1.0), 100, 150, 0.1).delta == 1.1000000000000001
    assert sparsim.micro_update_threshold(S(0.0), 10, 50, 0.1, 1e-12).delta == 1e-12
    assert sparsim.micro_update_threshold(S(0.0), 10, 3, 0.1).delta == 0.0
    with pytest.raises(ValueError):
        sparsim.micro_update_threshold(S(1.0), 10, 5, 1.0)
    rng = np.random.default_rng(11)
    for _ in range(500):
        d, a = float(rng.uniform(0, 10)), float(rng.uniform(0.001, 0.999))
        kt, ks = int(rng.integers(0, 1000)), int(rng.integers(0, 1000))
        assert sparsim.micro_update_threshold(S(d), kt, ks, a).delta == o.update_threshold(d, kt, ks, a)


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure mode")
def test_device_calls_fail_loudly_without_gpu(L):
    from paper_2310_00967_b200 import _lib
    cfg = _lib.micro_config()
    L.micro_config_default(C.byref(cfg))
    cfg.n_g = 1000
    h = C.c_void_p()
    rc = L.micro_ctx_create(C.byref(h), C.byref(cfg), None)
    assert rc == _lib.MICRO_ECUDA and not h.value
    assert L.micro_last_error()


def test_config_rejects_bad_gradient_types(L):
    """micro_config.grad_dtype: fp32 gradients need fp64 state and the MiCRO
    sparsifier; anything else is EINVAL before any device call (no GPU here)."""
    from paper_2310_00967_b200 import _lib
    cases = [(_lib.MICRO_F32, _lib.MICRO_GRAD_F32, 0), (_lib.MICRO_F64, 7, 0), (_lib.MICRO_F64, _lib.MICRO_GRAD_F32, 1)]
    for dtype, gd, kind in cases:
        cfg = _lib.micro_config()
        L.micro_config_default(C.byref(cfg))
        cfg.n_g, cfg.dtype, cfg.grad_dtype, cfg.sparsifier = 1000, dtype, gd, kind
        h = C.c_void_p()
        assert L.micro_ctx_create(C.byref(h), C.byref(cfg), None) == _lib.MICRO_EINVAL and not h.value
        assert b"gradient" in L.micro_last_error()


@pytest.mark.ref
def test_host_error_messages_match_the_reference(L):
    """The C ABI's status codes and messages are the reference's exceptions
    (tensor.hpp:49-55, sparsifier.cpp:73-75, :112-122), word for word."""
    from oracle import OracleError, Reference
    from paper_2310_00967_b200 import sparsim
    from paper_2310_00967_b200._lib import InvalidArgument
    ref = Reference()
    cases = [
        (lambda: sparsim.partition(3, 4, 0, 0), lambda: ref.partition(3, 4, 0, 0)),
        (lambda: sparsim.partition(8, 4, 0, 4), lambda: ref.partition(8, 4, 0, 4)),
        (lambda: sparsim.partition(8, 0, 0, 0), lambda: ref.partition(8, 0, 0, 0)),
        (lambda: sparsim.partition(8, 4, -1, 0), lambda: ref.partition(8, 4, -1, 0)),
        (lambda: sparsim.global_target_count(1.5, 100), lambda: ref.global_target_count(1.5, 100)),
        (lambda: sparsim.global_target_count(0.01, 0), lambda: ref.global_target_count(0.01, 0)),
        (lambda: sparsim.per_worker_target_count(0.01, 100, 0), lambda: ref.per_worker_target_count(0.01, 100, 0)),
        (lambda: sparsim.micro_update_threshold(sparsim.ThresholdState(1.0), 10, 5, 0.0),
         lambda: ref.update_threshold(1.0, 10, 5, 0.0)),
        (lambda: sparsim.micro_update_threshold(sparsim.ThresholdState(-1.0), 10, 5, 0.1),
         lambda: ref.update_threshold(-1.0, 10, 5, 0.1)),
    ]
    for ours, theirs in cases:
        with pytest.raises(InvalidArgument) as a:
            ours()
        with pytest.raises(OracleError) as b:
            theirs()
        theirs_msg = str(b.value).split("] ", 1)[-1]  # OracleError prefixes "[code] "
        assert str(a.value) == theirs_msg, (str(a.value), theirs_msg)
