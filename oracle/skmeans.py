"""Spherical k-means (sk-means) oracle — TEST INFRASTRUCTURE ONLY.

PAPER.md §4.2 "Spherical k-means (sk-means)" (lines 1133-1140): all points are projected to the
unit sphere before k-means runs, and proximity is the cosine similarity.  SPEC.md:353-360 fixes
the rest: rows normalised once up front; assignment by maximum cosine similarity, realised as the
Euclidean argmin on the unit sphere (for unit u, w: ||u - w||^2 = 2 (1 - u.w));
centroid update = mean, then re-normalised to unit length.  Readings (B6-B8): rows
are normalised in fp64 (squared norm summed in coordinate order, correctly rounded sqrt and
division) and rounded to fp32, the initial centroids likewise but kept in fp64; an empty cluster
keeps its centroid (A10), and so does a cluster whose mean is the zero vector.

Steps use the fp64 C oracle (``assign_brute``, ``cluster_sums``, ``update``); the normalisation is
written out here with numpy element-wise operations only (no reductions whose order numpy picks).
"""
from __future__ import annotations

import numpy as np

from .oracle import OracleResult, assign_brute, cluster_sums, sse, update


def _sq_norms(A):
    """sum_j A[:, j]^2 in coordinate order, fp64 (each square rounded, then added)."""
    ss = A[:, 0] * A[:, 0]
    for j in range(1, A.shape[1]):
        ss = ss + A[:, j] * A[:, j]
    return ss


def normalize_rows(X):
    """fp32 rows x / ||x|| ("every output row has unit L2 norm")."""
    X64 = np.asarray(X, dtype=np.float32).astype(np.float64)
    ss = _sq_norms(X64)
    if np.any(~(ss > 0)):
        raise ValueError("normalize_rows: zero row (domain error, SPEC.md:95)")
    return (X64 / np.sqrt(ss)[:, None]).astype(np.float32)


def normalize_centroids(C):
    """fp64 rows c / ||c|| (the initial centroids of sk-means)."""
    C = np.array(C, dtype=np.float64, copy=True)
    ss = _sq_norms(C)
    if np.any(~(ss > 0)):
        raise ValueError("normalize_centroids: zero centroid")
    return C / np.sqrt(ss)[:, None]


def renormalize(Cm, counts, Cold):
    """each non-empty cluster's mean re-normalised to unit length (in place);
    a zero mean keeps the previous centroid (reading B8)."""
    nz = np.asarray(counts) > 0
    ss = _sq_norms(Cm)
    ok = nz & (ss > 0)
    Cm[ok] = Cm[ok] / np.sqrt(ss[ok])[:, None]
    Cm[nz & ~(ss > 0)] = Cold[nz & ~(ss > 0)]
    return Cm


def skmeans(X, C0, max_iters, tol=0) -> OracleResult:
    """Brute-force sk-means from C0: Lloyd's loop (§4.1) on the unit sphere."""
    Xn = normalize_rows(X)
    n, d = Xn.shape
    C = normalize_centroids(np.asarray(C0, dtype=np.float64).reshape(-1, d))
    k = C.shape[0]
    a_prev = None
    changed, dists, empties, sses = [], [], [], []
    a = np.zeros(n, np.int32)
    for t in range(1, int(max_iters) + 1):
        a, _, _ = assign_brute(Xn, C)
        ch = n if a_prev is None else int((a != a_prev).sum())
        sums, counts = cluster_sums(Xn, a, k)
        Cm, empty = update(sums, counts, C)                 # mean, or the old centroid if empty
        C = renormalize(Cm, counts, C)
        changed.append(ch); dists.append(n * k); empties.append(empty)
        sses.append(sse(Xn, a, C))
        a_prev = a
        if ch <= tol:
            break
    T = len(changed)
    return OracleResult(a, C, T, np.array(changed, np.int64), np.array(dists, np.int64),
                        np.zeros(T, np.int64), np.array(empties, np.int32), np.array(sses))
