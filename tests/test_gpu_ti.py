"""GPU parity of the Elkan TI baseline (KM_PRUNE_TI, km_ti.cu) against the
oracle's mode=ti (oracle_ti_pass, reading B10): strict tier — assignments identical at every
iteration, centroids and SSE <= 1e-12 — plus the distance counts (soft 0.1 %: fp32 bounds with
directed rounding prune borderline candidates differently from fp64) and the paper's comparison
points: TI computes no more distances than MTI, and needs O(nk) memory."""
import json
import os

import numpy as np
import pytest

import oracle
from helpers import centroid_rel_err
from synth import make_config

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1902_09527_b200 import KMeans, KMeansError  # noqa: E402

HV = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "hand_vectors.json")))


def run(X, C0, iters, prune, per_iter=False):
    km = KMeans(torch.from_numpy(np.ascontiguousarray(X, np.float32)).cuda(), C0, prune=prune)
    a_hist = []
    if per_iter:
        it = 0
        for it in range(1, iters + 1):
            ch, _ = km.iterate()
            a_hist.append(km.assignments())
            if ch <= 0:
                break
        dists = None
    else:
        it, dists = km.run(iters, 0)
    out = dict(iterations=it, a=km.assignments(), C=km.centroids(), sse=km.sse(), stats=km.stats(),
               engine=km.engine, bytes=km.device_bytes, a_hist=a_hist, u=km.bounds())
    km.close()
    return out


def test_B2_ti_trace_on_gpu():
    e, e2 = HV["B2"], HV["B2_TI"]
    X = np.array(e["X"], np.float32)
    g = run(X, X[e["forgy"]].astype(float), 100, "ti")
    assert g["engine"] == "k_ti"
    assert g["iterations"] == e2["iterations"]
    assert [s["dists"] for s in g["stats"]] == e2["dists"]
    assert [s["changed"] for s in g["stats"]] == e2["changed"]
    assert [s["clause1"] for s in g["stats"]] == e2["clause1"]
    assert np.allclose(g["C"], np.array(e["C_T"], float), atol=1e-12, rtol=0)


@pytest.mark.parametrize("name,n,iters", [("c1", None, 100), ("c2", None, 50), ("c3", 2_000_000, 30),
                                          ("c4", 500_000, 30), ("c5", 200_000, 20)])
def test_ti_free_running_strict(name, n, iters):
    X, idx, _ = make_config(name, n=n)
    C0 = X[idx].astype(float)
    r = oracle.lloyd_trace(X, C0, iters, 0, "ti")
    hist = []
    oracle.lloyd_trace(X, C0, iters, 0, "brute", on_iter=lambda t, a, C, rec: hist.append(a.copy()))
    g = run(X, C0, iters, "ti", per_iter=True)
    assert g["iterations"] == r.iterations == len(hist)
    for t, (ag, ab) in enumerate(zip(g["a_hist"], hist), 1):
        assert np.array_equal(ag, ab), (t, int((ag != ab).sum()))
    assert np.array_equal(g["a"], r.a)
    assert centroid_rel_err(g["C"], r.C).max() <= 1e-12
    assert abs(g["sse"] - r.final_sse) <= 1e-12 * r.final_sse
    assert [s["changed"] for s in g["stats"]] == r.changed.tolist()
    gd = np.array([s["dists"] for s in g["stats"]])
    # soft check: 0.1 % relative, plus borderline rows (bound tests within the fp32 rounding margin
    # go either way; their number scales with n, not with the count: 1 per 100k rows)
    tol = 1e-3 * r.dists + 1e-5 * X.shape[0] + 2
    assert np.all(np.abs(gd - r.dists) <= tol), (gd.tolist(), r.dists.tolist())
    # TI's bounds only remove computations: fewer distances than MTI (same trajectory)
    m = run(X, C0, iters, "mti")
    md = np.array([s["dists"] for s in m["stats"]])
    assert np.all(gd <= md)
    # O(nk) memory of the lower-bound matrix
    k = C0.shape[0]
    assert g["bytes"] >= X.shape[0] * k * 4


def test_ti_bounds_sound_lockstep():
    """u >= ||x - C_used[a]|| after every TI pass (read through kmeans_get_bounds)."""
    X, idx, _ = make_config("c2")
    C0 = X[idx].astype(float)
    km = KMeans(torch.from_numpy(X).cuda(), C0, prune="ti")
    for _ in range(6):
        Cused = km.centroids()
        km.iterate()
        a = km.assignments()
        a_o, d1, _ = oracle.assign_brute(X, Cused)
        assert np.array_equal(a, a_o)
        u = km.bounds().astype(np.float64)
        assert np.all(u >= np.sqrt(d1) * (1 - 1e-14))
    km.close()


def test_ti_out_of_memory_is_reported():
    """C5-sized bounds (k = 1000, n = 100M: 400 GB) cannot fit: KM_ENOMEM, not a crash.  Here a
    k x n that exceeds the device's memory with a small point array (n rows of d = 1)."""
    free, total = torch.cuda.mem_get_info()
    k = 4096
    n = int(total // (4 * k)) + 1024
    X = torch.zeros((n, 1), dtype=torch.float32, device="cuda")
    X[:k, 0] = torch.arange(k, dtype=torch.float32, device="cuda")
    with pytest.raises(KMeansError, match="KM_ENOMEM"):
        KMeans(X, np.arange(k, dtype=np.float64).reshape(k, 1), prune="ti")
