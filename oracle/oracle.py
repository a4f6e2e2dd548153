"""ctypes wrapper over ``liboracle_kmeans.so`` (plain C, fp64, OpenMP) — TEST INFRASTRUCTURE ONLY.

Every function mirrors one C function in ``kmeans_oracle.c``; see that file's header for the
PAPER.md passages.  numpy is used only to hold arrays.
"""
from __future__ import annotations

import ctypes as ct
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle_kmeans.so")
_SRC = os.path.join(_HERE, "kmeans_oracle.c")


def build_oracle(force: bool = False) -> str:
    """Compile the oracle with gcc (-O2 -fopenmp, no fast-math, no FMA contraction)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               "-ffp-contract=off", "-o", _SO, _SRC])
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        build_oracle()
        L = ct.CDLL(_SO)
        P = ct.c_void_p
        i64, i32, dbl = ct.c_int64, ct.c_int32, ct.c_double
        L.oracle_assign_brute.argtypes = [P, i64, ct.c_int, P, ct.c_int, P, P, P]
        L.oracle_geometry.argtypes = [P, ct.c_int, ct.c_int, P, P]
        L.oracle_drift.argtypes = [P, P, ct.c_int, ct.c_int, P]
        L.oracle_cluster_sums.argtypes = [P, i64, ct.c_int, P, ct.c_int, ct.c_int, P, P]
        L.oracle_update.argtypes = [P, P, P, ct.c_int, ct.c_int, P]
        L.oracle_update.restype = ct.c_int
        L.oracle_sse.argtypes = [P, i64, ct.c_int, P, P]
        L.oracle_sse.restype = dbl
        L.oracle_mti_pass.argtypes = [P, i64, ct.c_int, P, ct.c_int, P, P, P, P, P, P]
        L.oracle_lloyd.argtypes = [P, i64, ct.c_int, ct.c_int, P, ct.c_int, i64, ct.c_int,
                                   ct.c_int, P, P, P, P, P, P, P, P]
        L.oracle_lloyd.restype = ct.c_int
        L.oracle_all_dists.argtypes = [P, i64, ct.c_int, P, ct.c_int, P]
        L.oracle_ti_pass.argtypes = [P, i64, ct.c_int, P, ct.c_int, P, P, P, P, P, P, P]
        L.oracle_num_threads.restype = ct.c_int
        L.oracle_set_threads.argtypes = [ct.c_int]
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ct.c_void_p)


def _X(X):
    X = np.ascontiguousarray(X, dtype=np.float32)
    if X.ndim == 1:
        X = X.reshape(-1, 1)
    return X


def _C(C, d=None):
    C = np.ascontiguousarray(C, dtype=np.float64)
    if C.ndim == 1:
        C = C.reshape(-1, 1 if d is None else d)
    return C


def num_threads() -> int:
    return lib().oracle_num_threads()


def set_threads(t: int) -> None:
    lib().oracle_set_threads(int(t))


def assign_brute(X, C):
    """(a int32[n], d1 fp64[n], d2 fp64[n]): argmin with lowest-index ties, best and
    second-best squared distances (Lloyd's assignment step)."""
    X = _X(X)
    n, d = X.shape
    C = _C(C, d)
    k = C.shape[0]
    a = np.empty(n, np.int32)
    d1 = np.empty(n, np.float64)
    d2 = np.empty(n, np.float64)
    lib().oracle_assign_brute(_p(X), n, d, _p(C), k, _p(a), _p(d1), _p(d2))
    return a, d1, d2


def geometry(C):
    """(H k x k, s k): H = 1/2 inter-centroid distances, s = min_{c'!=c} H (MTI, §3.3)."""
    C = _C(C)
    k, d = C.shape
    H = np.empty((k, k), np.float64)
    s = np.empty(k, np.float64)
    lib().oracle_geometry(_p(C), k, d, _p(H), _p(s))
    return H, s


def drift(Cnew, Cold):
    """f(c) = d(C_new[c], C_old[c])."""
    Cnew, Cold = _C(Cnew), _C(Cold)
    k, d = Cnew.shape
    f = np.empty(k, np.float64)
    lib().oracle_drift(_p(Cnew), _p(Cold), k, d, _p(f))
    return f


def cluster_sums(X, a, k, shards=1):
    """(sums k x d fp64, counts int64[k]) in fixed 64 Ki-row blocks (optionally sharded)."""
    X = _X(X)
    n, d = X.shape
    a = np.ascontiguousarray(a, dtype=np.int32)
    sums = np.empty((k, d), np.float64)
    counts = np.empty(k, np.int64)
    lib().oracle_cluster_sums(_p(X), n, d, _p(a), k, int(shards), _p(sums), _p(counts))
    return sums, counts


def update(sums, counts, Cold):
    """(C_new, #empty): mean of each cluster, previous centroid kept when empty (A10)."""
    Cold = _C(Cold)
    k, d = Cold.shape
    sums = _C(sums, d)
    counts = np.ascontiguousarray(counts, dtype=np.int64)
    Cnew = np.empty((k, d), np.float64)
    e = lib().oracle_update(_p(sums), _p(counts), _p(Cold), k, d, _p(Cnew))
    return Cnew, int(e)


def sse(X, a, C):
    """sum_i ||x_i - C[a_i]||^2 (Eq. 1, read as SSE)."""
    X = _X(X)
    n, d = X.shape
    C = _C(C, d)
    a = np.ascontiguousarray(a, dtype=np.int32)
    return float(lib().oracle_sse(_p(X), n, d, _p(a), _p(C)))


def mti_pass(X, C, Cprev, a, u):
    """One MTI pass (t >= 2) with centroids C (previous pass used Cprev): returns
    (a_new, u_new, dists, clause1, changed).  Inputs are not modified."""
    X = _X(X)
    n, d = X.shape
    C, Cprev = _C(C, d), _C(Cprev, d)
    k = C.shape[0]
    H, s = geometry(C)
    f = drift(C, Cprev)
    a2 = np.array(a, dtype=np.int32, copy=True)
    u2 = np.array(u, dtype=np.float64, copy=True)
    o3 = np.zeros(3, np.int64)
    lib().oracle_mti_pass(_p(X), n, d, _p(C), k, _p(H), _p(s), _p(f), _p(a2), _p(u2), _p(o3))
    return a2, u2, int(o3[0]), int(o3[1]), int(o3[2])


def all_dists(X, C):
    """n x k fp64 matrix of ||x_i - C[c]|| (Elkan's lower bounds after iteration 1)."""
    X = _X(X)
    n, d = X.shape
    C = _C(C, d)
    L = np.empty((n, C.shape[0]), np.float64)
    lib().oracle_all_dists(_p(X), n, d, _p(C), C.shape[0], _p(L))
    return L


def ti_pass(X, C, Cprev, a, u, L):
    """One Elkan TI pass (t >= 2; kmeans_oracle.c oracle_ti_pass) with centroids C (previous pass
    used Cprev): returns (a_new, u_new, L_new, dists, clause1, changed).  Inputs are not modified."""
    X = _X(X)
    n, d = X.shape
    C, Cprev = _C(C, d), _C(Cprev, d)
    k = C.shape[0]
    H, s = geometry(C)
    f = drift(C, Cprev)
    a2 = np.array(a, dtype=np.int32, copy=True)
    u2 = np.array(u, dtype=np.float64, copy=True)
    L2 = np.array(L, dtype=np.float64, copy=True).reshape(n, k)
    o3 = np.zeros(3, np.int64)
    lib().oracle_ti_pass(_p(X), n, d, _p(C), k, _p(H), _p(s), _p(f), _p(a2), _p(u2), _p(L2), _p(o3))
    return a2, u2, L2, int(o3[0]), int(o3[1]), int(o3[2])


@dataclass
class OracleResult:
    a: np.ndarray
    C: np.ndarray
    iterations: int
    changed: np.ndarray = field(repr=False)
    dists: np.ndarray = field(repr=False)
    clause1: np.ndarray = field(repr=False)
    empty: np.ndarray = field(repr=False)
    sse: np.ndarray = field(repr=False)

    @property
    def dists_total(self) -> int:
        return int(self.dists.sum())

    @property
    def final_sse(self) -> float:
        return float(self.sse[-1]) if self.sse.size else float("nan")


def lloyd(X, C0, max_iters, tol=0, mode="brute", shards=1, with_sse=True) -> OracleResult:
    """Full Lloyd's run from C0 (§4.1), brute force or MTI (§3.3); see kmeans_oracle.c."""
    X = _X(X)
    n, d = X.shape
    C0 = _C(C0, d)
    k = C0.shape[0]
    m = {"brute": 0, "mti": 1, "ti": 2}[mode]
    a = np.zeros(n, np.int32)
    C = np.empty((k, d), np.float64)
    it = np.zeros(1, np.int32)
    cap = max(1, int(max_iters))
    ch = np.zeros(cap, np.int64)
    ds = np.zeros(cap, np.int64)
    c1 = np.zeros(cap, np.int64)
    em = np.zeros(cap, np.int32)
    ss = np.zeros(cap, np.float64) if with_sse else None
    rc = lib().oracle_lloyd(_p(X), n, d, k, _p(C0), int(max_iters), int(tol), m, int(shards),
                            _p(a), _p(C), _p(it), _p(ch), _p(ds), _p(c1), _p(em), _p(ss))
    if rc == -2:
        raise MemoryError("oracle_lloyd: TI lower-bound matrix (n x k fp64) could not be allocated")
    if rc != 0:
        raise ValueError("oracle_lloyd: usage error (n<1, d<1, k<1, k>n or max_iters<0)")
    T = int(it[0])
    return OracleResult(a, C, T, ch[:T], ds[:T], c1[:T], em[:T],
                        ss[:T] if ss is not None else np.zeros(0))


def lloyd_trace(X, C0, max_iters, tol=0, mode="mti", on_iter=None) -> OracleResult:
    """The loop of ``oracle_lloyd`` (kmeans_oracle.c) driven step by step from Python over the
    same C primitives, so that a caller can observe every iteration: ``on_iter(t, a_t, C_t,
    record)`` is called after iteration t's update (a_t: this pass's assignments, C_t: the means
    it produced; record: dict of changed/dists/clause1/empty/sse).  Same steps, same order:
    iteration 1 brute force (u = exact distance; TI: every distance as lower bounds), then
    brute force, one MTI pass or one Elkan TI pass
    (geometry/drift of the centroids this pass uses, §3.3), block-ordered sums, update with
    reading A10, SSE w.r.t. (C_t, a_t), stop iff changed <= tol (§4.1).  Pinned to
    ``lloyd`` (bitwise) by tests/test_oracle_trace.py."""
    X = _X(X)
    n, d = X.shape
    C = _C(C0, d).copy()
    k = C.shape[0]
    if n < 1 or k < 1 or k > n or max_iters < 0:
        raise ValueError("lloyd_trace: usage error")
    Cprev = C.copy()
    a = np.zeros(n, np.int32)
    u = L = None
    recs = []
    t = 0
    for t in range(1, max_iters + 1):
        clause1 = 0
        if t == 1 or mode == "brute":
            aprev = a
            a, d1, _ = assign_brute(X, C)
            dists = n * k
            changed = n if t == 1 else int(np.count_nonzero(a != aprev))
            if mode in ("mti", "ti"):
                u = np.sqrt(d1)
            if mode == "ti":
                L = all_dists(X, C)
        elif mode == "ti":
            a, u, L, dists, clause1, changed = ti_pass(X, C, Cprev, a, u, L)
        else:
            a, u, dists, clause1, changed = mti_pass(X, C, Cprev, a, u)
        sums, counts = cluster_sums(X, a, k)
        Cprev = C
        C, empty = update(sums, counts, Cprev)
        rec = dict(t=t, changed=int(changed), dists=int(dists), clause1=int(clause1),
                   empty=int(empty), sse=sse(X, a, C))
        recs.append(rec)
        if on_iter is not None:
            on_iter(t, a, C, rec)
        if changed <= tol:
            break
    T = len(recs)
    col = lambda key, dt: np.array([r[key] for r in recs], dt)  # noqa: E731
    return OracleResult(a, C, T, col("changed", np.int64), col("dists", np.int64),
                        col("clause1", np.int64), col("empty", np.int32), col("sse", np.float64))
