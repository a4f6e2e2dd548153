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


def _fraction_draw(D2, u):
    """Eq. 2 with reading B9 in exact rationals: the first i with sum_{j<=i} D2_j > u * sum D2."""
    from fractions import Fraction
    vals = [Fraction(float(v)) for v in D2]
    target = Fraction(float(u)) * sum(vals)
    run = Fraction(0)
    for i, v in enumerate(vals):
        run += v
        if run > target:
            return i
    return -1


def test_draw_equals_exact_rational_definition():
    """Rows with D² over a wide exponent range (and zeros), many u: the oracle's integer sums
    pick the row the exact rational definition picks."""
    rng = np.random.default_rng(1)
    for trial in range(40):
        n = int(rng.integers(1, 300))
        D2 = rng.random(n) * np.exp2(rng.integers(-60, 60, n).astype(float))
        D2[rng.random(n) < 0.2] = 0.0
        if not (D2 > 0).any():
            D2[0] = 1.0
        for u in [0.0, float(rng.random()), float(rng.random()), np.nextafter(1.0, 0.0)]:
            assert oracle.kmeanspp.draw(D2, u) == _fraction_draw(D2, u), (trial, u)


def test_draw_is_exact_where_fp64_sums_are_not():
    """D² = (2^53, 1, 1): the fp64 total rounds to 2^53, but the exact one is 2^53 + 2; with the
    largest u below 1 the exact target 2^53 + 1 - 2^-52 is crossed first by row 1 (an fp64
    running-sum implementation would answer row 0)."""
    D2 = np.array([2.0 ** 53, 1.0, 1.0])
    u = float(np.nextafter(1.0, 0.0))
    assert oracle.kmeanspp.draw(D2, u) == 1
    assert oracle.kmeanspp.draw(np.array([1.0, 2.0, 3.0]), 0.5) == 2                 # P = 3 is not > 3
    assert oracle.kmeanspp.draw(np.array([1.0, 2.0, 3.0]), float(np.nextafter(0.5, 0.0))) == 1
    assert oracle.kmeanspp.draw(np.array([0.0, 0.0, 5.0, 0.0]), 0.0) == 2             # zeros never drawn


def test_large_array_matches_cumsum():
    """Two million rows: the exact draw agrees with an fp64 cumulative sum up to its rounding."""
    rng = np.random.default_rng(1)
    n = 2 * 1024 * 1024 + 3 * 1024 + 123
    D2 = rng.random(n) ** 4
    tot = np.cumsum(D2)
    for u in [0.0, 0.1, 0.3333, 0.5, 0.77, 0.999999]:
        i = oracle.kmeanspp.draw(D2, u)
        j = int(np.searchsorted(tot, u * tot[-1], side="right"))
        assert abs(i - j) <= 1, (u, i, j)


def test_multirun_hand_case():
    """PAPER.md §4.3 best-of-r, hand-checked.  Rectangle (0,0), (0,1), (4,0), (4,1), k = 2, first
    row 0, D² = (0, 1, 16, 17), total 34.  Run A (u = 0.01, target 0.34): row 1 -> centres
    (0,0), (0,1) -> Lloyd's fixed point {(0,0),(4,0)} / {(0,1),(4,1)}: C = (2,0), (2,1), SSE 16.
    Run B (u = 0.5, target 17): row 3 -> centres (0,0), (4,1) -> {(0,0),(0,1)} / {(4,0),(4,1)}:
    C = (0,0.5), (4,0.5), SSE 1.  The best of (A, B) is B; of (B, A) it is B again (index 0);
    of (A, A) the first."""
    X = np.array([[0, 0], [0, 1], [4, 0], [4, 1]], np.float32)
    A, B = (0, [0.01]), (0, [0.5])
    i, a, C, sse, it = oracle.kmeanspp_multirun(X, 2, [A, B], 20)
    assert i == 1 and sse == 1.0 and C.tolist() == [[0.0, 0.5], [4.0, 0.5]] and a.tolist() == [0, 0, 1, 1]
    i, _, _, sse, _ = oracle.kmeanspp_multirun(X, 2, [B, A], 20)
    assert i == 0 and sse == 1.0
    i, a, C, sse, _ = oracle.kmeanspp_multirun(X, 2, [A, A], 20)
    assert i == 0 and sse == 16.0 and C.tolist() == [[2.0, 0.0], [2.0, 1.0]] and a.tolist() == [0, 1, 0, 1]


def test_multirun_keeps_min_sse():
    """PAPER.md §4.3: the best of r runs is the one with the minimum SSE."""
    rng = np.random.default_rng(2)
    X = np.concatenate([rng.normal(size=(200, 2)) + c for c in ([0, 0], [8, 0], [0, 8])]).astype(np.float32)
    runs = [(int(rng.integers(600)), rng.random(2)) for _ in range(4)]
    best = oracle.kmeanspp_multirun(X, 3, runs, 50)
    sses = [oracle.lloyd(X, oracle.seed_plusplus(X, 3, u, f)[1], 50, 0, "brute").final_sse for f, u in runs]
    assert best[0] == int(np.argmin(sses)) and best[3] == min(sses)
