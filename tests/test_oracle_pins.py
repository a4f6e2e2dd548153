"""Pins for the fp64 CPU oracle (``oracle/``) against values the paper, SPEC worked examples,
hand-checked traces, closed forms and the mathematics fix — never against the oracle itself.

Each test names the passage it pins.  All run on CPU (``-m "not gpu"``).
"""
import itertools
import json
import math
import os

import numpy as np
import pytest

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")
HV = json.load(open(os.path.join(GOLD, "hand_vectors.json")))


# ---- SPEC worked examples -------------------------------
def test_euclid_examples():
    for x, c, dist in HV["spec_euclid"]:
        a, d1, d2 = oracle.assign_brute(np.array([x], np.float32), np.array([c], np.float64))
        assert a[0] == 0 and math.sqrt(d1[0]) == dist and d2[0] == math.inf


def test_sse_example():
    e = HV["spec_sse"]
    assert oracle.sse(np.array(e["X"], np.float32), np.zeros(2, np.int32), np.array(e["C"])) == e["sse"]


@pytest.mark.parametrize("shards", [1, 2])
def test_reduce_example(shards):
    e = HV["spec_reduce"]
    sums, counts = oracle.cluster_sums(np.array(e["X"], np.float32), np.zeros(2, np.int32), 1, shards)
    C, empty = oracle.update(sums, counts, np.zeros((1, 2)))
    assert empty == 0 and np.array_equal(C, np.array(e["C"], float)) and counts[0] == 2


def test_geometry_example_and_k1():
    e = HV["spec_geometry"]
    H, s = oracle.geometry(np.array(e["C"], float))
    assert np.array_equal(H, np.array(e["H"], float)) and np.array_equal(s, np.array(e["s"], float))
    H1, s1 = oracle.geometry(np.array([[3.0, 4.0]]))
    assert s1[0] == math.inf and H1[0, 0] == 0.0


def test_drift_inflate_example():
    # u = 1.0, drift 0.5 -> 1.5 (drift = d(C_new, C_old))
    f = oracle.drift(np.array([[0.0, 0.5]]), np.array([[0.0, 0.0]]))
    assert f[0] == 0.5 and 1.0 + f[0] == 1.5


# ---- hand-checked traces --------------------------------------------
@pytest.mark.parametrize("mode", ["brute", "mti", "ti"])
def test_B1_one_dim(mode):
    e = HV["B1"]
    r = oracle.lloyd(np.array(e["X"], np.float32), np.array(e["C0"], float), 100, 0, mode)
    assert r.iterations == e["iterations"]
    assert r.a.tolist() == e["a_T"]
    assert np.array_equal(r.C, np.array(e["C_T"], float))
    assert r.final_sse == e["sse"]
    assert r.changed.tolist() == e["changed"]
    assert r.dists.tolist() == e[mode + "_dists"]


def test_B2_mti_trace():
    e = HV["B2"]
    X = np.array(e["X"], np.float32)
    C0 = X[e["forgy"]].astype(float)
    r = oracle.lloyd(X, C0, 100, 0, "mti")
    assert r.iterations == e["iterations"]
    assert r.dists.tolist() == e["dists"]
    assert r.changed.tolist() == e["changed"]
    assert r.clause1.tolist() == e["clause1"]
    assert np.allclose(r.C, np.array(e["C_T"], float), rtol=0, atol=1e-12)
    assert abs(r.final_sse - e["sse"]) < 1e-9
    assert abs(r.sse[0] - e["sse_1"]) < 1e-9
    assert r.dists_total == e["dists_total"]
    rb = oracle.lloyd(X, C0, 100, 0, "brute")
    assert rb.dists_total == e["brute_dists_total"] and rb.a.tolist() == r.a.tolist()
    # iteration-1 state: C_1 and u_1 (u = exact distance to the assigned centroid)
    r1 = oracle.lloyd(X, C0, 1, 0, "mti")
    assert np.allclose(r1.C, np.array(e["C_1"], float), atol=1e-12)
    a1, d1, _ = oracle.assign_brute(X, C0)
    assert np.allclose(np.sqrt(d1), e["u_1"], atol=1e-12)


def test_B2_ti_trace():
    """Elkan TI (reading B10) on the B2 data: the hand-checked trace and the per-point state
    (assignments, upper bounds, n x k lower bounds) after iteration 2."""
    e, e2 = HV["B2"], HV["B2_TI"]
    X = np.array(e["X"], np.float32)
    C0 = X[e["forgy"]].astype(float)
    r = oracle.lloyd(X, C0, 100, 0, "ti")
    assert r.iterations == e2["iterations"] and r.dists.tolist() == e2["dists"]
    assert r.changed.tolist() == e2["changed"] and r.clause1.tolist() == e2["clause1"]
    assert np.allclose(r.C, np.array(e["C_T"], float), rtol=0, atol=1e-12)
    assert abs(r.final_sse - e["sse"]) < 1e-9 and r.dists_total == e2["dists_total"]
    a1, d1, _ = oracle.assign_brute(X, C0)
    L1 = oracle.all_dists(X, C0)
    assert np.allclose(L1, np.abs(X.astype(float) - C0.ravel()[None, :]), atol=1e-12)
    C1 = np.array(e["C_1"], float)
    a2, u2, L2, dists, c1, ch = oracle.ti_pass(X, C1, C0, a1, np.sqrt(d1), L1)
    st = e2["state_2"]
    assert a2.tolist() == st["a"] and (dists, c1, ch) == (st["dists"], st["clause1"], st["changed"])
    assert np.allclose(u2, st["u"], atol=1e-12) and np.allclose(L2, np.array(st["L"], float), atol=1e-12)


def test_B3_half_factor():
    """The literal clause (no 1/2) would keep x in a; with Elkan's 1/2 it moves (A1)."""
    e = HV["B3"]
    C = np.array(e["C"], float)
    X = np.array([e["x"]], np.float32)
    a, u, dists, c1, changed = oracle.mti_pass(X, C, C, [e["a"]], [e["u"]])
    assert a[0] == e["a_new"] and u[0] == e["u_new"] and dists == e["dists"] and c1 == 0 and changed == 1
    # the literal (unsound) clause 1 would have pruned: u <= min d(a, .) = 2
    assert e["u"] <= np.linalg.norm(C[0] - C[1])


@pytest.mark.parametrize("mode", ["brute", "mti", "ti"])
def test_B5_empty_cluster(mode):
    e = HV["B5"]
    X = np.array(e["X"], np.float32)
    C0 = X[e["forgy"]].astype(float)
    r1 = oracle.lloyd(X, C0, 1, 0, mode)
    assert r1.a.tolist() == e["a_1"] and np.allclose(r1.C, np.array(e["C_1"], float), atol=1e-12)
    r = oracle.lloyd(X, C0, 100, 0, mode)
    assert r.iterations == e["iterations"]
    assert r.a.tolist() == e["a_T"]
    assert np.allclose(r.C, np.array(e["C_T"], float), atol=1e-12)
    assert r.empty.tolist() == e["empty"]
    assert abs(r.final_sse - e["sse"]) < 1e-12


def test_max_iters_zero():
    # max_iters = 0 returns the initial centroids and zero iterations
    X = np.array([[0.0], [1.0], [5.0]], np.float32)
    C0 = np.array([[0.0], [5.0]])
    r = oracle.lloyd(X, C0, 0)
    assert r.iterations == 0 and np.array_equal(r.C, C0)


def test_usage_errors():
    with pytest.raises(ValueError):
        oracle.lloyd(np.zeros((2, 1), np.float32), np.zeros((3, 1)), 5)   # k > n


# ---- closed forms / special cases ----------------------------------------------------------
@pytest.mark.parametrize("mode", ["brute", "mti", "ti"])
def test_k1_global_mean(mode):
    rng = np.random.default_rng(5)
    X = rng.normal(size=(257, 3)).astype(np.float32)
    r = oracle.lloyd(X, X[:1].astype(float), 10, 0, mode)
    mean = np.array([math.fsum(float(v) for v in X[:, j]) / 257 for j in range(3)])
    assert r.iterations == 2 and np.allclose(r.C[0], mean, rtol=0, atol=1e-14)
    if mode != "brute":   # s = +inf: every point is clause-1 from iteration 2
        assert r.dists.tolist() == [257, 0] and r.clause1.tolist() == [0, 257]


@pytest.mark.parametrize("mode", ["brute", "mti", "ti"])
def test_k_equals_n(mode):
    X = np.array([[0, 0], [1, 0], [0, 3], [7, 7], [2, 9]], np.float32)
    r = oracle.lloyd(X, X.astype(float), 10, 0, mode)
    assert r.sse[0] == 0.0 and r.a.tolist() == [0, 1, 2, 3, 4] and r.iterations == 2


# ---- global optimum on tiny inputs (brute-force enumeration, pinned by the 1-D DP) ----------
def _partitions(n, k):
    """All set partitions of range(n) into exactly k blocks (restricted growth strings)."""
    def rec(i, labels, m):
        if i == n:
            if m == k:
                yield list(labels)
            return
        for c in range(min(m + 1, k)):
            if n - i - 1 < k - max(m, c + 1):
                continue
            labels.append(c)
            yield from rec(i + 1, labels, max(m, c + 1))
            labels.pop()
    yield from rec(0, [], 0)


def _part_sse(X, labels, k):
    X = X.astype(float)
    lab = np.asarray(labels)
    s = 0.0
    for c in range(k):
        P = X[lab == c]
        s += ((P - P.mean(axis=0)) ** 2).sum()
    return s


def _opt_enum(X, k):
    best, arg = math.inf, None
    for lab in _partitions(len(X), k):
        v = _part_sse(X, lab, k)
        if v < best:
            best, arg = v, lab
    return best, arg


def _opt_dp_1d(x, k):
    """Textbook O(k n^2) DP: the optimal 1-D k-means partition is contiguous in sorted order."""
    x = np.sort(np.asarray(x, float))
    n = len(x)

    def cost(i, j):  # x[i..j] inclusive
        seg = x[i:j + 1]
        return float(((seg - seg.mean()) ** 2).sum())
    D = np.full((k + 1, n + 1), math.inf)
    D[0, 0] = 0.0
    for m in range(1, k + 1):
        for j in range(1, n + 1):
            D[m, j] = min((D[m - 1, i] + cost(i, j - 1) for i in range(m - 1, j)), default=math.inf)
    return D[k, n]


def test_partition_enumerator_counts():
    # Stirling numbers of the second kind: S(6,3)=90, S(7,2)=63, S(8,4)=1701
    assert sum(1 for _ in _partitions(6, 3)) == 90
    assert sum(1 for _ in _partitions(7, 2)) == 63
    assert sum(1 for _ in _partitions(8, 4)) == 1701


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_enumerator_matches_1d_dp(seed):
    x = np.random.default_rng(seed).normal(size=9).astype(np.float32)
    e, _ = _opt_enum(x.reshape(-1, 1), 3)
    assert abs(e - _opt_dp_1d(x, 3)) < 1e-12


@pytest.mark.parametrize("seed,n,k,d", [(0, 9, 3, 2), (1, 10, 3, 2), (2, 8, 4, 3), (3, 12, 3, 2)])
def test_lloyd_vs_global_optimum(seed, n, k, d):
    X = np.random.default_rng(seed).normal(size=(n, d)).astype(np.float32)
    opt, lab = _opt_enum(X, k)
    for mode in ("brute", "mti", "ti"):
        for idx in itertools.combinations(range(n), k):
            r = oracle.lloyd(X, X[list(idx)].astype(float), 100, 0, mode)
            assert r.final_sse >= opt - 1e-9
    # Lloyd from the optimal partition's centroids is a fixed point with SSE_opt
    lab = np.asarray(lab)
    Copt = np.stack([X[lab == c].astype(float).mean(axis=0) for c in range(k)])
    for mode in ("brute", "mti", "ti"):
        r = oracle.lloyd(X, Copt, 100, 0, mode)
        assert r.changed[-1] == 0 and r.iterations == 2
        assert abs(r.final_sse - opt) <= 1e-12 * max(1.0, opt)
        assert np.allclose(r.C, Copt, atol=1e-12)


# ---- invariants: MTI losslessness, bound soundness, SSE monotone, dists <= n k --------------
def _mixture(seed, n, d, K, spread=8.0):
    rng = np.random.default_rng(seed)
    means = rng.uniform(-spread, spread, (K, d))
    lab = rng.integers(0, K, n)
    return (means[lab] + rng.normal(size=(n, d))).astype(np.float32)


@pytest.mark.parametrize("seed,n,d,k", [(0, 3000, 4, 8), (1, 5000, 8, 20), (2, 2000, 3, 50), (3, 4000, 16, 12)])
def test_mti_lossless_and_monotone(seed, n, d, k):
    X = _mixture(seed, n, d, max(2, k // 2))
    idx = np.random.default_rng(seed + 100).choice(n, k, replace=False)
    C0 = X[idx].astype(float)
    rb = oracle.lloyd(X, C0, 60, 0, "brute")
    rm = oracle.lloyd(X, C0, 60, 0, "mti")
    assert rb.iterations == rm.iterations
    assert np.array_equal(rb.a, rm.a) and np.array_equal(rb.C, rm.C)
    assert np.array_equal(rb.changed, rm.changed) and np.array_equal(rb.sse, rm.sse)
    assert np.all(rm.dists <= n * k) and rm.dists[0] == n * k and np.all(rm.dists >= 0)
    assert rm.dists_total < rb.dists_total
    assert np.all(np.diff(rb.sse) <= 1e-12 * rb.sse[:-1])
    # per-iteration lockstep losslessness and bound soundness of the MTI pass
    a, _, _ = oracle.assign_brute(X, C0)
    C_prev = C0
    sums, counts = oracle.cluster_sums(X, a, k)
    C, _ = oracle.update(sums, counts, C0)
    u = np.sqrt(oracle.assign_brute(X, C0)[1])
    for t in range(2, 8):
        am, um, dists, c1, ch = oracle.mti_pass(X, C, C_prev, a, u)
        ab, d1, _ = oracle.assign_brute(X, C)
        assert np.array_equal(am, ab)
        true = np.sqrt(((X.astype(float) - C[am]) ** 2).sum(axis=1))
        assert np.all(um >= true * (1 - 1e-15))
        assert 0 <= dists <= n * k and c1 <= n
        sums, counts = oracle.cluster_sums(X, am, k)
        C_prev, (C, _) = C, oracle.update(sums, counts, C)
        a, u = am, um


@pytest.mark.parametrize("seed,n,d,k", [(0, 3000, 4, 8), (1, 5000, 8, 20), (2, 2000, 3, 50), (3, 4000, 16, 12)])
def test_ti_lossless_sound_and_fewer_dists_than_mti(seed, n, d, k):
    """Elkan TI (reading B10): identical assignments/centroids to brute force at every
    iteration, sound bounds after every pass (u >= d(x, C[a]), l[c] <= d(x, C[c]) for every c),
    and never more distances than MTI in the same iteration (TI's extra bounds only
    remove computations)."""
    X = _mixture(seed, n, d, max(2, k // 2))
    idx = np.random.default_rng(seed + 100).choice(n, k, replace=False)
    C0 = X[idx].astype(float)
    rb = oracle.lloyd(X, C0, 60, 0, "brute")
    rm = oracle.lloyd(X, C0, 60, 0, "mti")
    rt = oracle.lloyd(X, C0, 60, 0, "ti")
    assert rt.iterations == rb.iterations
    assert np.array_equal(rt.a, rb.a) and np.array_equal(rt.C, rb.C) and np.array_equal(rt.changed, rb.changed)
    assert rt.dists[0] == n * k and np.all(rt.dists <= rm.dists) and np.all(rt.dists >= 0)
    a, d1, _ = oracle.assign_brute(X, C0)
    u, L = np.sqrt(d1), oracle.all_dists(X, C0)
    sums, counts = oracle.cluster_sums(X, a, k)
    C_prev, (C, _) = C0, oracle.update(sums, counts, C0)
    Xd = X.astype(float)
    for t in range(2, 8):
        at, ut, Lt, dists, c1, ch = oracle.ti_pass(X, C, C_prev, a, u, L)
        ab, _, _ = oracle.assign_brute(X, C)
        assert np.array_equal(at, ab)
        true = np.sqrt(((Xd[:, None, :] - C[None, :, :]) ** 2).sum(axis=2))
        assert np.all(Lt <= true * (1 + 1e-15))
        assert np.all(ut >= true[np.arange(n), at] * (1 - 1e-15))
        sums, counts = oracle.cluster_sums(X, at, k)
        C_prev, (C, _) = C, oracle.update(sums, counts, C)
        a, u, L = at, ut, Lt


def test_sharded_equals_unsharded():
    X = _mixture(7, 200_000, 8, 10)
    a, _, _ = oracle.assign_brute(X, X[:10].astype(float))
    s1, c1 = oracle.cluster_sums(X, a, 10, 1)
    for G in (2, 3, 8):
        sg, cg = oracle.cluster_sums(X, a, 10, G)
        assert np.array_equal(c1, cg)
        assert np.max(np.abs(sg - s1) / np.maximum(np.abs(s1), 1e-300)) <= 1e-13
    r1 = oracle.lloyd(X, X[:10].astype(float), 20, 0, "mti", shards=1)
    r8 = oracle.lloyd(X, X[:10].astype(float), 20, 0, "mti", shards=8)
    assert np.array_equal(r1.a, r8.a) and r1.iterations == r8.iterations
    assert np.max(np.abs(r1.C - r8.C)) <= 1e-13 * np.max(np.abs(r1.C))


def test_thread_count_determinism():
    X = _mixture(9, 150_000, 4, 6)
    C0 = X[:6].astype(float)
    t0 = oracle.num_threads()
    try:
        oracle.set_threads(1)
        r1 = oracle.lloyd(X, C0, 15, 0, "mti")
        oracle.set_threads(max(2, t0))
        r2 = oracle.lloyd(X, C0, 15, 0, "mti")
    finally:
        oracle.set_threads(t0)
    assert np.array_equal(r1.C, r2.C) and np.array_equal(r1.a, r2.a) and np.array_equal(r1.sse, r2.sse)
