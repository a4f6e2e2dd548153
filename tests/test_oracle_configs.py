"""Oracle on the seeded configs: library cross-check (scikit-learn Lloyd) and the
independent golden trajectories of SURVEY.md Appendix C; synthetic-recipe hashes."""
import json
import os

import numpy as np
import pytest

import oracle
from synth import CONFIGS, make_config, sha256_points

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "appendix_c.json")))


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_synth_hash_and_forgy(name):
    X, idx, man = make_config(name)
    assert X.shape == (CONFIGS[name].n, CONFIGS[name].d) and X.dtype == np.float32
    assert sha256_points(X) == GOLD["sha256"][name]
    assert idx[:8].tolist() == GOLD["forgy_head"][name]
    assert len(set(idx.tolist())) == CONFIGS[name].k


def test_synth_worker_independence():
    a = make_config("c1", workers=1)[0]
    b = make_config("c1", workers=4)[0]
    assert np.array_equal(a, b)
    s1 = make_config("c3", n=3_000_000, workers=1)[0]
    s4 = make_config("c3", n=3_000_000, workers=4)[0]
    assert np.array_equal(s1, s4)


def _check_traj(r, g, rtol_sse=1e-10):
    assert r.iterations == g["iterations"]
    assert r.changed[:6].tolist() == g["changed_head"]
    assert r.changed[-3:].tolist() == g["changed_tail"]
    assert int(r.empty[-1]) == g["empty"]
    assert abs(r.final_sse - g["sse"]) <= rtol_sse * g["sse"] + 1e-3
    assert abs(np.abs(r.C).sum() - g["sum_abs_C"]) <= 1e-9 * g["sum_abs_C"] + 1e-7
    sizes = np.bincount(r.a, minlength=r.C.shape[0])
    assert sizes.min() == g["sizes_min"] and sizes.max() == g["sizes_max"]


@pytest.mark.parametrize("mode", ["brute", "mti"])
def test_c1_golden_trajectory(mode):
    X, idx, _ = make_config("c1")
    r = oracle.lloyd(X, X[idx].astype(float), CONFIGS["c1"].max_iters, 0, mode)
    _check_traj(r, GOLD["trajectory"]["c1"])


def test_c1_scikit_learn_lloyd():
    sk = pytest.importorskip("sklearn.cluster")
    X, idx, _ = make_config("c1")
    C0 = X[idx].astype(np.float64)
    km = sk.KMeans(n_clusters=10, init=C0, n_init=1, max_iter=100, tol=0.0,
                   algorithm="lloyd").fit(X.astype(np.float64))
    r = oracle.lloyd(X, C0, 100, 0, "brute")
    # converged, empty-free run: sklearn's relabel-at-end and empty relocation do not apply
    assert km.n_iter_ == r.iterations
    rel = np.linalg.norm(km.cluster_centers_ - r.C, axis=1) / np.linalg.norm(r.C, axis=1)
    assert rel.max() <= 1e-12
    assert np.array_equal(km.labels_, r.a)


def test_c2_golden_trajectory_mti():
    X, idx, _ = make_config("c2")
    r = oracle.lloyd(X, X[idx].astype(float), CONFIGS["c2"].max_iters, 0, "mti")
    _check_traj(r, GOLD["trajectory"]["c2"])
    assert np.all(np.diff(r.sse) <= 1e-12 * r.sse[:-1])
