"""Pins for the k-means++ seeding oracle (``oracle/kmeanspp.py``; Eq. 2)
against closed-form draws on tiny inputs and the sampling law itself."""
import numpy as np
import pytest

import oracle


def test_three_points_closed_form():
    """1-D {0, 1, 10}, c1 = 0: D² = (0, 1, 100), total 101 -> u < 1/101 picks 1, else 10."""
    X = np.array([[0], [1], [10]], np.float32)
    for u, want in [(0.0, 1), (0.5 / 101, 1), (0.99 / 101, 1), (1.01 / 101, 2), (0.5, 2), (0.999, 2)]:
        ch, C = oracle.seed_plusplus(X, 2, [u], 0)
        assert ch.tolist() == [0, want] and C[1, 0] == float(X[want, 0])


def test_chosen_row_is_never_redrawn():
    """A chosen row has D = 0, so its probability is 0 (Eq. 2)."""
    X = np.array([[0, 0], [3, 4], [6, 8], [0, 5]], np.float32)
    ch, _ = oracle.seed_plusplus(X, 4, [0.3, 0.6, 0.9], 1)
    assert sorted(ch.tolist()) == [0, 1, 2, 3]


def test_k1_and_duplicates():
    X = np.array([[1, 1], [1, 1], [1, 1]], np.float32)
    ch, C = oracle.seed_plusplus(X, 1, [], 2)
    assert ch.tolist() == [2] and C.tolist() == [[1.0, 1.0]]
    with pytest.raises(ValueError):                    # every D² is 0: no second centre
        oracle.seed_plusplus(X, 2, [0.5], 0)


def test_draw_law_matches_d2_weights():
    """Over a grid of uniforms the draw frequencies equal D² / Σ D² (Eq. 2) to grid resolution."""
    rng = np.random.default_rng(0)
    X = rng.normal(size=(12, 3)).astype(np.float32)
    D2 = oracle.kmeanspp.d2_to(X.astype(np.float64), X[0].astype(np.float64))
    counts = np.zeros(12)
    us = (np.arange(20000) + 0.5) / 20000
    for u in us:
        counts[oracle.kmeanspp.draw(D2, u)] += 1
    assert np.allclose(counts / len(us), D2 / D2.sum(), atol=1e-4)


def test_block_boundaries():
    """Rows spread over several blocks and groups: the draw lands where the cumulative weight
    crosses u·total (brute-force cumulative sum over all rows)."""
    rng = np.random.default_rng(1)
    n = 2 * 1024 * 1024 + 3 * 1024 + 123
    D2 = rng.random(n) ** 4
    tot = np.cumsum(D2)
    for u in [0.0, 0.1, 0.3333, 0.5, 0.77, 0.999999]:
        i = oracle.kmeanspp.draw(D2, u)
        j = int(np.searchsorted(tot, u * tot[-1], side="right"))
        assert abs(i - j) <= 1, (u, i, j)       # equal up to fp64 rounding of the two sums


def test_multirun_keeps_min_sse():
    """PAPER.md §4.3: the best of r runs is the one with the minimum SSE."""
    rng = np.random.default_rng(2)
    X = np.concatenate([rng.normal(size=(200, 2)) + c for c in ([0, 0], [8, 0], [0, 8])]).astype(np.float32)
    runs = [(int(rng.integers(600)), rng.random(2)) for _ in range(4)]
    best = oracle.kmeanspp_multirun(X, 3, runs, 50)
    sses = [oracle.lloyd(X, oracle.seed_plusplus(X, 3, u, f)[1], 50, 0, "brute").final_sse for f, u in runs]
    assert best[0] == int(np.argmin(sses)) and best[3] == min(sses)
