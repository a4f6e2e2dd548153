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

BLOCK = 65536


def d2_to(X64, c):
    """Σ_j (x_j - c_j)² per row, fp64, coordinate order (each difference and square rounded)."""
    s = np.zeros(X64.shape[0])
    for j in range(X64.shape[1]):
        t = X64[:, j] - c[j]
        s = s + t * t
    return s


def _running_sum(vals):
    """Running sums of vals in order (np.add.accumulate is a sequential left-to-right loop)."""
    return np.add.accumulate(vals) if len(vals) else np.zeros(0)


def draw(D2, u):
    """The row drawn for uniform u (reading B9); -1 if every D² is 0."""
    n = D2.shape[0]
    nb = (n + BLOCK - 1) // BLOCK
    bsum = [float(_running_sum(D2[b * BLOCK:(b + 1) * BLOCK])[-1]) for b in range(nb)]
    total = 0.0
    for v in bsum:
        total = total + v
    target = u * total
    R, bs, Rs = 0.0, -1, 0.0
    for b in range(nb):
        nxt = R + bsum[b]
        if nxt > target:
            bs, Rs = b, R
            break
        R = nxt
    scan = True
    if bs < 0:                                   # rounding left target >= total
        scan = False
        pos = [b for b in range(nb) if bsum[b] > 0.0]
        if not pos:
            return -1
        bs = pos[-1]
    t2 = target - Rs
    blk = D2[bs * BLOCK:(bs + 1) * BLOCK]
    run = _running_sum(blk)
    last = -1
    for i in range(blk.shape[0]):
        if blk[i] > 0.0:
            last = bs * BLOCK + i
            if scan and run[i] > t2:
                return bs * BLOCK + i
    return last


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
