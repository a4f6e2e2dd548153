"""k-means++ D² seeding oracle — TEST INFRASTRUCTURE ONLY.

PAPER.md §4.3 "k-means++" (lines 1141-1159), Eq. 2: each new centroid is drawn from the data
with probability D(v)² / Σ_v D(v)², D(v) = the distance of v to the nearest centroid already
chosen.  Reading B9 makes the draw reproducible and exact: the caller supplies
the first index and the k-1 uniforms; D² is summed in fp64 over the coordinates in order; the
total is formed over fixed blocks of 65536 rows (each summed in row order, the block sums added
in block order); the chosen row is the first row of the first block whose running block sum
exceeds u·total, whose in-block running sum exceeds u·total minus the preceding blocks' sum,
and whose D² is positive.  Written as plain loops: slow, obviously in order.
"""
from __future__ import annotations

import numpy as np

BLOCK = 1024        # rows per block
GROUP = 1024        # blocks per group


def d2_to(X64, c):
    """Σ_j (x_j - c_j)² per row, fp64, coordinate order (each difference and square rounded)."""
    s = np.zeros(X64.shape[0])
    for j in range(X64.shape[1]):
        t = X64[:, j] - c[j]
        s = s + t * t
    return s


def _seq_sum(vals):
    """Left-to-right sum (np.add.accumulate is a sequential loop); 0.0 for an empty list."""
    return float(np.add.accumulate(vals)[-1]) if len(vals) else 0.0


def _first_crossing(vals, t):
    """Index of the first running sum (left to right) that exceeds t, with that sum's start
    value; (-1, _) if none."""
    run = 0.0
    for i, v in enumerate(vals):
        nxt = run + v
        if nxt > t:
            return i, run
        run = nxt
    return -1, run


def _last_positive(vals):
    pos = np.nonzero(np.asarray(vals) > 0.0)[0]
    return int(pos[-1]) if pos.size else -1


def draw(D2, u):
    """The row drawn for uniform u (reading B9); -1 if every D² is 0.

    Order of every sum: rows of a block (BLOCK rows) in row order; blocks of a group (GROUP
    blocks) in block order; groups in group order.  The target u·total is located by running
    sums at each level, top-down; where rounding leaves no crossing, the last positive entry."""
    n = D2.shape[0]
    nb = (n + BLOCK - 1) // BLOCK
    ng = (nb + GROUP - 1) // GROUP
    bsum = [_seq_sum(D2[b * BLOCK:(b + 1) * BLOCK]) for b in range(nb)]
    gsum = [_seq_sum(bsum[g * GROUP:(g + 1) * GROUP]) for g in range(ng)]
    total = _seq_sum(gsum)
    target = u * total
    g, R = _first_crossing(gsum, target)
    scan = g >= 0
    if not scan:
        g = _last_positive(gsum)
        if g < 0:
            return -1
    gb = bsum[g * GROUP:(g + 1) * GROUP]
    if scan:
        t1 = target - R
        bi, P = _first_crossing(gb, t1)
        scan = bi >= 0
    if not scan:
        bi = _last_positive(gb)
    b = g * GROUP + bi
    blk = D2[b * BLOCK:(b + 1) * BLOCK]
    if scan:
        t2 = t1 - P
        run = 0.0
        for i in range(blk.shape[0]):
            run = run + blk[i]
            if blk[i] > 0.0 and run > t2:
                return b * BLOCK + i
    return b * BLOCK + _last_positive(blk)


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
    """PAPER.md §4.3: r seeded runs of Lloyd's, the one with the smallest SSE (earlier on ties)."""
    from .oracle import lloyd
    best = None
    for i, (first, u) in enumerate(runs):
        _, C0 = seed_plusplus(X, k, u, first)
        r = lloyd(X, C0, max_iters, tol, "brute")
        if best is None or r.final_sse < best[3]:
            best = (i, r.a, r.C, r.final_sse, r.iterations)
    return best
