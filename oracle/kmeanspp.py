"""k-means++ D² seeding oracle — TEST INFRASTRUCTURE ONLY (only tests/, smoke() and bench.py's
cpu_baseline may import it; the product path never does).

PAPER.md §4.3 "k-means++" (lines 1141-1159), Eq. 2: each new centroid is drawn from the data
with probability D(v)² / Σ_v D(v)², D(v) = the distance of v to the nearest centroid already
chosen.  Reading B9 makes the draw reproducible and exact:

* the caller supplies the first index and the k-1 uniforms u ∈ [0, 1);
* D(v)² is the fp64 value Σ_j (x_j - c_j)² computed in coordinate order (each difference,
  square and addition rounded to nearest), minimised over the chosen centres;
* the drawn row is the FIRST row i whose exact prefix sum Σ_{j<=i} D_j² exceeds u · Σ_j D_j²,
  prefix, total and product taken exactly (real arithmetic on the fp64 values).

The exact sums are Python integers: every D² is a multiple of 2^-350 (differences of fp32
values are multiples of 2^-149, so their squares and the rounded sums of squares are multiples
of 2^-298 rounded to 53 bits), so D² · 2^350 is an exact integer.  Written as plain loops over
the rows: slow, obviously the definition.  Nothing here mirrors the GPU's blocking.
"""
from __future__ import annotations

from itertools import accumulate

import numpy as np

SCALE_BITS = 350           # D² * 2^SCALE_BITS is an integer for every D² (see above)


def d2_to(X64, c):
    """Σ_j (x_j - c_j)² per row, fp64, coordinate order (each difference and square rounded)."""
    s = np.zeros(X64.shape[0])
    for j in range(X64.shape[1]):
        t = X64[:, j] - c[j]
        s = s + t * t
    return s


def _exact_int(v: float) -> int:
    """v * 2^SCALE_BITS as an exact integer (v >= 0 a multiple of 2^-SCALE_BITS)."""
    m, e = float(v).as_integer_ratio()          # v = m / e exactly, e a power of two
    q, r = divmod(m << SCALE_BITS, e)
    if r:
        raise ValueError(f"D² {v!r} is not a multiple of 2^-{SCALE_BITS}")
    return q


def draw(D2, u):
    """The row drawn for uniform u (reading B9): the first i with exact Σ_{j<=i} D² > u Σ D²;
    -1 if every D² is 0.  u·total is exact: u = mu / 2^s, so P_i > u·T <=> P_i > floor(mu·T / 2^s)
    for integer P_i."""
    ints = [_exact_int(v) for v in np.asarray(D2, np.float64).tolist()]
    prefix = list(accumulate(ints))
    total = prefix[-1] if prefix else 0
    if total == 0:
        return -1
    mu, den = float(u).as_integer_ratio()       # u = mu / den, den = 2^s
    target = (mu * total) // den
    for i, p in enumerate(prefix):               # first crossing (always exists: u < 1)
        if p > target:
            return i
    raise AssertionError("no crossing with u < 1")


def seed_plusplus(X, k, uniforms, first_index):
    """(chosen int64[k], centroids fp64 k x d) — Eq. 2 with reading B9."""
    X64 = np.asarray(X, dtype=np.float32).astype(np.float64)
    chosen = [int(first_index)]
    D2 = d2_to(X64, X64[first_index])
    for m in range(1, k):
        i = draw(D2, float(uniforms[m - 1]))
        if i < 0:
            raise ValueError("fewer than k distinct rows")
        chosen.append(i)
        D2 = np.minimum(D2, d2_to(X64, X64[i]))
    return np.array(chosen, np.int64), X64[chosen].copy()


def kmeanspp_multirun(X, k, runs, max_iters, tol=0):
    """PAPER.md §4.3: r seeded runs of Lloyd's, the one with the smallest SSE (the earliest on
    ties).  Returns (index, a, C, sse, iterations) of the kept run."""
    from .oracle import lloyd
    best = None
    for i, (first, u) in enumerate(runs):
        _, C0 = seed_plusplus(X, k, u, first)
        r = lloyd(X, C0, max_iters, tol, "brute")
        if best is None or r.final_sse < best[3]:
            best = (i, r.a, r.C, r.final_sse, r.iterations)
    return best
