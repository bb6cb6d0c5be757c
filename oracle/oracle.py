"""ctypes faces of the CHECKERS — test infrastructure only.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
reference arm may import this module.  The product path
(``paper_2310_00967_b200``) never does.

* :class:`Oracle` — ``_build/libmicro_oracle.so``, the C restatement
  (``micro_oracle.c``) in float32 (the GPU contract) and float64.
* :class:`Reference` — ``_ref/libsparsim_ref.so``, the reference's own
  hot-path translation units compiled verbatim (``ref_driver.cpp``).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libmicro_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libsparsim_ref.so")
REPORT_SO = os.path.join(HERE, "_ref", "libsparsim_report.so")

i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
I64, U64, I32, U32, DBL = C.c_int64, C.c_uint64, C.c_int, C.c_uint32, C.c_double


class OracleError(Exception):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code
        self.msg = msg


def build() -> None:
    """Build the checkers (idempotent).  The reference arm only when the
    reference sources are present (this container)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _load(path: str) -> C.CDLL:
    if not os.path.exists(path):
        build()
    return C.CDLL(path)


class Oracle:
    def __init__(self):
        L = self.lib = _load(ORACLE_SO)
        L.orc_last_error.restype = C.c_char_p
        L.orc_partition.argtypes = [I64, I32, I64, I32, C.POINTER(I64), C.POINTER(I64)]
        L.orc_global_target_count.argtypes = [DBL, I64, C.POINTER(U64)]
        L.orc_per_worker_target_count.argtypes = [DBL, I64, I32, I32, C.POINTER(U64)]
        L.orc_update_threshold.argtypes = [C.POINTER(DBL), U64, U64, DBL, DBL]
        L.orc_gaussian.argtypes = [U64, U32, U64, I64, f32p]
        L.orc_gaussian.restype = None
        for suf, fp in (("f32", f32p), ("f64", f64p)):
            getattr(L, f"orc_select_{suf}").argtypes = [fp, I64, I64, I64, DBL, i64p, fp, C.POINTER(I64)]
            getattr(L, f"orc_all_reduce_sparse_values_{suf}").argtypes = [fp, I32, I64, i64p, I64, fp]
            getattr(L, f"orc_step_{suf}").argtypes = [
                I64, I32, DBL, DBL, DBL, I32, I32, I64, DBL, fp, fp, f64p, C.c_void_p,
                i64p, C.c_void_p, C.c_void_p, C.POINTER(I64), f64p]
            getattr(L, f"orc_fetch_union_{suf}").argtypes = [i64p, fp, I64]

    def _check(self, rc):
        if rc:
            raise OracleError(rc, self.lib.orc_last_error().decode())

    def partition(self, n_g, n, t, worker):
        s, e = I64(), I64()
        self._check(self.lib.orc_partition(n_g, n, t, worker, C.byref(s), C.byref(e)))
        return s.value, e.value

    def global_target_count(self, d, n_g):
        k = U64()
        self._check(self.lib.orc_global_target_count(d, n_g, C.byref(k)))
        return k.value

    def per_worker_target_count(self, d, n_g, n, full=False):
        k = U64()
        self._check(self.lib.orc_per_worker_target_count(d, n_g, n, int(full), C.byref(k)))
        return k.value

    def update_threshold(self, delta, k_target, k_selected, alpha, min_threshold=1e-12):
        d = DBL(delta)
        self._check(self.lib.orc_update_threshold(C.byref(d), k_target, k_selected, alpha, min_threshold))
        return d.value

    def gaussian(self, seed, worker, t, n):
        out = np.empty(n, np.float32)
        self.lib.orc_gaussian(seed, worker, t, n, out)
        return out

    def select(self, acc, start, end, delta):
        acc = np.ascontiguousarray(acc)
        suf = "f32" if acc.dtype == np.float32 else "f64"
        m = max(end - start, 0)
        idx = np.empty(m, np.int64)
        val = np.empty(m, acc.dtype)
        cnt = I64()
        self._check(getattr(self.lib, f"orc_select_{suf}")(acc, acc.size, start, end, delta, idx, val, C.byref(cnt)))
        return idx[: cnt.value].copy(), val[: cnt.value].copy()

    def all_reduce_sparse_values(self, accs, union_idx):
        accs = np.ascontiguousarray(accs)
        suf = "f32" if accs.dtype == np.float32 else "f64"
        n, n_g = accs.shape
        u = np.ascontiguousarray(union_idx, np.int64)
        out = np.empty(u.size, accs.dtype)
        self._check(getattr(self.lib, f"orc_all_reduce_sparse_values_{suf}")(accs, n, n_g, u, u.size, out))
        return out


class OracleCluster:
    """n in-process workers stepped by ``orc_step_{f32,f64}`` (harness.cpp:121-224)."""

    def __init__(self, n_g, n, density=0.01, delta0=0.01, alpha=0.01, min_threshold=1e-12,
                 full=False, error_feedback=True, dtype=np.float32, model=False):
        self.o = Oracle()
        self.n_g, self.n = n_g, n
        self.cfg = (density, alpha, min_threshold, int(full), int(error_feedback))
        self.dtype = np.dtype(dtype)
        self.e = np.zeros((n, n_g), self.dtype)
        self.delta = np.full(n, delta0, np.float64)
        self.x = np.zeros(n_g, self.dtype) if model else None
        suf = "f32" if self.dtype == np.float32 else "f64"
        self.fn = getattr(self.o.lib, "orc_step_" + suf)
        self.fetch = getattr(self.o.lib, "orc_fetch_union_" + suf)

    def step(self, G, eta, t):
        G = np.ascontiguousarray(G, self.dtype).reshape(self.n, self.n_g)
        counts = np.empty(self.n, np.int64)
        K = I64()
        dused = np.empty(self.n, np.float64)
        d, a, eps, full, ef = self.cfg
        xp = self.x.ctypes.data if self.x is not None else None
        # the union stays inside the oracle (sized to it) and is fetched at its size
        rc = self.fn(self.n_g, self.n, d, a, eps, full, ef, t, eta, self.e, G, self.delta, xp,
                     counts, None, None, C.byref(K), dused)
        if rc:
            raise OracleError(rc, self.o.lib.orc_last_error().decode())
        uidx = np.empty(K.value, np.int64)
        usum = np.empty(K.value, self.dtype)
        self.fetch(uidx, usum, K.value)
        return dict(counts=counts, union_idx=uidx, union_sum=usum,
                    delta_used=dused, delta_next=self.delta.copy())


class Reference:
    """The reference's own code (oracle/_ref/libsparsim_ref.so), fp64."""

    def __init__(self):
        if not os.path.exists(REF_SO):
            build()
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(f"{REF_SO} missing: build it where /root/reference exists")
        L = self.lib = C.CDLL(REF_SO)
        L.ref_last_error.restype = C.c_char_p
        L.ref_partition.argtypes = [I64, I32, I64, I32, C.POINTER(I64), C.POINTER(I64)]
        L.ref_global_target_count.argtypes = [DBL, I64, C.POINTER(U64)]
        L.ref_per_worker_target_count.argtypes = [DBL, I64, I32, I32, C.POINTER(U64)]
        L.ref_update_threshold.argtypes = [C.POINTER(DBL), U64, U64, DBL, DBL]
        L.ref_select_by_threshold.argtypes = [f64p, I64, I64, I64, DBL, i64p, f64p, C.POINTER(I64)]
        L.ref_accumulate.argtypes = [f64p, I64, DBL, f64p, I64, f64p]
        L.ref_compensate.argtypes = [f64p, I64, i64p, I64, f64p]
        L.ref_all_gather_indices.argtypes = [I32, i64p, i64p, i64p, C.POINTER(I64), C.POINTER(U64)]
        L.ref_all_reduce_sparse_values.argtypes = [f64p, I32, I64, i64p, I64, f64p]
        L.ref_all_reduce_sparse.argtypes = [f64p, I32, I64, i64p, I64, f64p]
        L.ref_error_metric.argtypes = [f64p, I32, I64, C.POINTER(DBL)]
        L.ref_cluster_create.argtypes = [I64, I32, DBL, DBL, DBL, DBL, I32, I32]
        L.ref_cluster_create.restype = C.c_void_p
        L.ref_cluster_destroy.argtypes = [C.c_void_p]
        L.ref_cluster_destroy.restype = None
        L.ref_cluster_step.argtypes = [C.c_void_p, f64p, DBL, I64, C.c_void_p, i64p, i64p, f64p,
                                       C.POINTER(I64), f64p]
        L.ref_cluster_residual.argtypes = [C.c_void_p, I32, f64p]
        L.ref_cluster_thresholds.argtypes = [C.c_void_p, f64p]
        L.ref_cluster_set_options.argtypes = [C.c_void_p, I32, I32]
        L.ref_cluster_set_state.argtypes = [C.c_void_p, I32, f64p, DBL]
        L.ref_cluster_dense.argtypes = [C.c_void_p, f64p]
        L.ref_cluster_phase_times.argtypes = [C.c_void_p, f64p]
        L.ref_cluster_phase_times.restype = None
        L.ref_cluster_step_kind.argtypes = [C.c_void_p, I32, f64p, DBL, I64, C.c_void_p, i64p, i64p, f64p,
                                            C.POINTER(I64)]

    def _check(self, rc):
        if rc:
            raise OracleError(rc, self.lib.ref_last_error().decode())

    def partition(self, n_g, n, t, worker):
        s, e = I64(), I64()
        self._check(self.lib.ref_partition(n_g, n, t, worker, C.byref(s), C.byref(e)))
        return s.value, e.value

    def global_target_count(self, d, n_g):
        k = U64()
        self._check(self.lib.ref_global_target_count(d, n_g, C.byref(k)))
        return k.value

    def per_worker_target_count(self, d, n_g, n, full=False):
        k = U64()
        self._check(self.lib.ref_per_worker_target_count(d, n_g, n, int(full), C.byref(k)))
        return k.value

    def update_threshold(self, delta, k_target, k_selected, alpha, min_threshold=1e-12):
        d = DBL(delta)
        self._check(self.lib.ref_update_threshold(C.byref(d), k_target, k_selected, alpha, min_threshold))
        return d.value

    def select_by_threshold(self, acc, start, end, delta):
        acc = np.ascontiguousarray(acc, np.float64)
        m = max(end - start, 0)
        idx = np.empty(max(m, 1), np.int64)
        val = np.empty(max(m, 1), np.float64)
        cnt = I64()
        self._check(self.lib.ref_select_by_threshold(acc, acc.size, start, end, delta, idx, val, C.byref(cnt)))
        return idx[: cnt.value].copy(), val[: cnt.value].copy()

    def accumulate(self, e, eta, g):
        e = np.ascontiguousarray(e, np.float64)
        g = np.ascontiguousarray(g, np.float64)
        out = np.empty(max(e.size, g.size), np.float64)
        self._check(self.lib.ref_accumulate(e, e.size, eta, g, g.size, out))
        return out

    def compensate(self, acc, sel):
        acc = np.ascontiguousarray(acc, np.float64)
        sel = np.ascontiguousarray(sel, np.int64)
        out = np.empty(acc.size, np.float64)
        self._check(self.lib.ref_compensate(acc, acc.size, sel if sel.size else np.zeros(1, np.int64), sel.size, out))
        return out

    def all_gather_indices(self, selections):
        counts = np.array([len(s) for s in selections], np.int64)
        concat = np.ascontiguousarray(np.concatenate([np.asarray(s, np.int64) for s in selections])
                                      if len(selections) else np.zeros(0, np.int64))
        out = np.empty(max(concat.size, 1), np.int64)
        K, tot = I64(), U64()
        self._check(self.lib.ref_all_gather_indices(len(selections), counts,
                                                    concat if concat.size else np.zeros(1, np.int64),
                                                    out, C.byref(K), C.byref(tot)))
        return out[: K.value].copy(), counts, tot.value

    def all_reduce_sparse_values(self, accs, union_idx):
        accs = np.ascontiguousarray(accs, np.float64)
        n, n_g = accs.shape
        u = np.ascontiguousarray(union_idx, np.int64)
        out = np.empty(max(u.size, 1), np.float64)
        self._check(self.lib.ref_all_reduce_sparse_values(accs, n, n_g, u if u.size else np.zeros(1, np.int64),
                                                          u.size, out))
        return out[: u.size].copy()

    def all_reduce_sparse(self, accs, union_idx):
        accs = np.ascontiguousarray(accs, np.float64)
        n, n_g = accs.shape
        u = np.ascontiguousarray(union_idx, np.int64)
        out = np.empty(n_g, np.float64)
        self._check(self.lib.ref_all_reduce_sparse(accs, n, n_g, u if u.size else np.zeros(1, np.int64),
                                                   u.size, out))
        return out

    def error_metric(self, residuals):
        r = np.ascontiguousarray(residuals, np.float64)
        out = DBL()
        n = r.shape[0] if r.ndim == 2 else 0
        self._check(self.lib.ref_error_metric(r if r.size else np.zeros(1), n, r.shape[-1] if r.ndim == 2 else 0,
                                              C.byref(out)))
        return out.value


class RefCluster:
    """run_iteration's MiCRO branch over the reference's own functions (fp64)."""

    def __init__(self, n_g, n, density=0.01, delta0=0.01, alpha=0.01, min_threshold=1e-12,
                 full=False, error_feedback=True, model=False):
        self.r = Reference()
        self.n_g, self.n = n_g, n
        self.h = self.r.lib.ref_cluster_create(n_g, n, density, delta0, alpha, min_threshold,
                                               int(full), int(error_feedback))
        if not self.h:
            raise OracleError(1, self.r.lib.ref_last_error().decode())
        self.x = np.zeros(n_g, np.float64) if model else None

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            self.r.lib.ref_cluster_destroy(h)
            self.h = None

    KINDS = {"micro": 0, "topk": 1, "cltk": 2, "hard": 3, "dense": 4}

    def step(self, G, eta, t, kind="micro"):
        G = np.ascontiguousarray(G, np.float64).reshape(self.n, self.n_g)
        counts = np.empty(self.n, np.int64)
        uidx = np.empty(self.n_g, np.int64)
        usum = np.empty(self.n_g, np.float64)
        K = I64()
        xp = self.x.ctypes.data if self.x is not None else None
        if kind != "micro":  # harness.cpp:152-181
            self.r._check(self.r.lib.ref_cluster_step_kind(self.h, self.KINDS[kind], G, eta, t, xp, counts, uidx,
                                                           usum, C.byref(K)))
            return dict(counts=counts, union_idx=uidx[: K.value].copy(), union_sum=usum[: K.value].copy())
        dused = np.empty(self.n, np.float64)
        self.r._check(self.r.lib.ref_cluster_step(self.h, G, eta, t, xp, counts, uidx, usum, C.byref(K), dused))
        dn = np.empty(self.n, np.float64)
        self.r.lib.ref_cluster_thresholds(self.h, dn)
        return dict(counts=counts, union_idx=uidx[: K.value].copy(), union_sum=usum[: K.value].copy(),
                    delta_used=dused, delta_next=dn)

    def set_options(self, dense=False, threads=1):
        """dense: also form all_reduce_sparse(...) / n each step; threads: run
        the per-worker loops on that many host threads."""
        self.r.lib.ref_cluster_set_options(self.h, int(dense), int(threads))

    def set_state(self, i, residual, delta):
        self.r._check(self.r.lib.ref_cluster_set_state(self.h, i, np.ascontiguousarray(residual, np.float64),
                                                       float(delta)))

    def dense(self):
        out = np.empty(self.n_g, np.float64)
        self.r._check(self.r.lib.ref_cluster_dense(self.h, out))
        return out

    def residual(self, i):
        out = np.empty(self.n_g, np.float64)
        self.r._check(self.r.lib.ref_cluster_residual(self.h, i, out))
        return out

    def residuals(self):
        return np.stack([self.residual(i) for i in range(self.n)])

    def phase_times(self):
        out = np.empty(4, np.float64)
        self.r.lib.ref_cluster_phase_times(self.h, out)
        return out


class ReferenceReport:
    """The reference's own record writer (report.cpp, oracle/_ref/libsparsim_report.so)."""

    TASKS = {"quadratic": 0, "logreg": 1, "mlp2": 2}
    KINDS = {"micro": 0, "topk": 1, "cltk": 2, "hard": 3, "dense": 4}
    FIELDS = ("actual_density", "buildup_factor", "redundant_traffic_factor", "error_norm", "threshold",
              "loss", "time_grad", "time_select", "time_comm", "time_overhead")

    def __init__(self):
        if not os.path.exists(REPORT_SO):
            build()
        if not os.path.exists(REPORT_SO):
            raise FileNotFoundError(f"{REPORT_SO} missing: build it where /root/reference exists")
        self.lib = C.CDLL(REPORT_SO)
        self.lib.ref_emit.argtypes = [I32, C.c_char_p, i64p, f64p, I64, i64p, f64p]

    def emit(self, fmt: str, path: str, records, cfg: dict) -> None:
        t = np.array([r["t"] for r in records] or [0], np.int64)
        cols = np.array([[float(r.get(f, 0.0)) for f in self.FIELDS] for r in records] or [[0.0] * 10], np.float64)
        ints = np.array([cfg["workers"], cfg["iterations"], cfg["batch_size"], cfg["seed"], self.TASKS[cfg["task"]],
                         cfg["dimension"], cfg["samples"], 0 if cfg["per_worker_k"] == "split" else 1,
                         cfg["decay_at"], int(cfg["error_feedback"]), self.KINDS[cfg["sparsifier"]]], np.int64)
        dbls = np.array([cfg["density"], cfg["delta0"], cfg["alpha"], cfg["eps_delta"], cfg["lr"], cfg["decay_factor"],
                         cfg["latency_per_collective"], cfg["bytes_per_element"], cfg["bandwidth"],
                         cfg["compute_time_per_op"]], np.float64)
        rc = self.lib.ref_emit(0 if fmt == "csv" else 1, path.encode(), t, np.ascontiguousarray(cols), len(records),
                               ints, dbls)
        if rc:
            raise OracleError(rc, "ref_emit failed")


class BaselineCluster:
    """TEST INFRASTRUCTURE: numpy restatement of run_iteration's comparison
    sparsifiers (harness.cpp:152-224) in the fp32 contract (or fp64, where it
    is pinned bit for bit to the reference's own code by
    tests/test_oracle_baselines.py):
      topk   select_topk (sparsifier.cpp:39-67): k_global largest |acc| over the
             whole vector, tie -> lower index, ascending
      cltk   cltk_select (sparsifier.cpp:85-97): the leader t mod n only
      hard   hard_threshold_select (sparsifier.cpp:99-101): |acc| > delta0
      dense  select_all (sparsifier.cpp:103-108)
    then the union (sorted unique), worker-order sums from +0, x -= s/n and
    the union zeroed on every worker (EF off: everything)."""

    def __init__(self, n_g, n, kind, density=0.01, delta0=0.01, error_feedback=True, dtype=np.float32,
                 model=False):
        self.n_g, self.n, self.kind = n_g, n, kind
        self.dtype = np.dtype(dtype)
        self.delta0 = delta0
        self.ef = error_feedback
        self.k = Oracle().global_target_count(density, n_g)
        self.e = np.zeros((n, n_g), self.dtype)
        self.x = np.zeros(n_g, self.dtype) if model else None

    def _topk(self, a):
        k = min(self.k, a.size)
        mag = np.abs(a)
        order = np.lexsort((np.arange(a.size), -mag))  # |acc| descending, then index ascending
        return np.sort(order[:k])

    def step(self, G, eta, t):
        G = np.asarray(G).reshape(self.n, self.n_g).astype(self.dtype)
        if not np.all(np.isfinite(G)):
            raise OracleError(3, "non-finite gradient")
        acc = self.e + self.dtype.type(eta) * G  # two roundings, like e + eta*G
        sels = [np.empty(0, np.int64) for _ in range(self.n)]
        if self.kind == "topk":
            sels = [self._topk(acc[i]) for i in range(self.n)]
        elif self.kind == "cltk":
            sels[t % self.n] = self._topk(acc[t % self.n])
        elif self.kind == "hard":
            sels = [np.flatnonzero(np.abs(acc[i]).astype(np.float64) > self.delta0) for i in range(self.n)]
        elif self.kind == "dense":
            sels = [np.arange(self.n_g) for _ in range(self.n)]
        else:
            raise ValueError(self.kind)
        union = np.unique(np.concatenate(sels)).astype(np.int64)
        s = np.zeros(union.size, self.dtype)
        for r in range(self.n):  # worker order from +0 (collectives.cpp:44-45)
            s = s + acc[r][union]
        if self.x is not None:
            self.x[union] = self.x[union] - s / self.dtype.type(self.n)
        acc[:, union] = 0
        if not self.ef:
            acc[:] = 0
        self.e = acc
        return dict(counts=np.array([x.size for x in sels], np.int64), union_idx=union, union_sum=s)
