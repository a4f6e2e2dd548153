"""Full BASELINE-size parity: C3, C4 and C5 free-running through the whole trajectory against the
oracle's golden trajectories (tests/golden/traj_<cfg>.json, written by tools/make_golden.py from
oracle.lloyd_trace in MTI mode — validated lossless against brute force — and synth/ only).

Every iteration t (the engine and launch configuration bench.py times):
  * a_t bit-exact: sha256 of the GPU's assignment vector (caller order) == the oracle's;
  * C_t <= 1e-12 per-centroid relative (strict tier; the BASELINE tier is 1e-5);
  * changed_t and empty_t exact; SSE_t <= 1e-12 relative; iteration counts equal;
  * dists_t within 0.1 % of the oracle's MTI count (soft check of SURVEY §8(c): fp32 bounds with
    directed rounding decide borderline prunes differently); clause1 within 0.1 % of n.
At two iterations, independently of the golden file: the sampled rows' assignments equal the
fp64 brute-force argmin over the centroids the pass used (§4.1, 1104-1112), and the
MTI bounds read back through kmeans_get_bounds are sound, u_i >= ||x_i - C_used[a_i]||
(§3.3, 1026-1034).
"""
import hashlib
import json
import os

import numpy as np
import pytest

import oracle
from helpers import centroid_rel_err
from synth import CONFIGS, make_config, sha256_points

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1902_09527_b200 import KMeans  # noqa: E402

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, np.int32).tobytes()).hexdigest()


def _independent_checks(X, a, u, Cused, rng, m):
    rows = np.sort(rng.choice(X.shape[0], m, replace=False))
    a_o, d1, _ = oracle.assign_brute(X[rows], Cused)
    assert int((a[rows] != a_o).sum()) == 0
    diff = X[rows].astype(np.float64) - Cused[a[rows]]
    dist = np.sqrt(np.einsum("ij,ij->i", diff, diff))
    bad = u[rows].astype(np.float64) < dist * (1 - 1e-14)
    assert not bad.any(), int(bad.sum())


@pytest.mark.parametrize("engine", ["cuda", "screen", "tensor_screen", "tensor_chunked"])
@pytest.mark.parametrize("name", ["c3", "c4", "c5"])
def test_full_size_trajectory(name, engine):
    path = os.path.join(GOLD, f"traj_{name}.json")
    if not os.path.exists(path):
        pytest.fail(f"missing golden trajectory {path} (tools/make_golden.py {name})")
    g = json.load(open(path))
    Cg = np.load(os.path.join(GOLD, f"traj_{name}_C.npy"))
    asamp = np.load(os.path.join(GOLD, f"traj_{name}_asample.npy"))
    spec = CONFIGS[name]
    X, idx, _ = make_config(name)
    assert X.shape == (spec.n, spec.d)
    assert sha256_points(X) == g["sha256_X"], "synthetic input differs from the golden run's"
    C0 = X[idx].astype(np.float64)
    km = KMeans(torch.from_numpy(X).cuda(), C0, prune="mti", engine=engine)
    assert km.engine == {"cuda": "k_walk", "screen": "k_screen", "tensor_screen": "k_mti_tc_screen", "tensor_chunked": "k_tcc"}[engine]
    rng = np.random.default_rng(101)
    T = g["iterations"]
    check_at = {2, T}
    t = 0
    for t in range(1, spec.max_iters + 1):
        Cused = km.centroids()
        changed, dists = km.iterate()
        rec = g["per_iter"][t - 1]
        a = km.assignments()
        if _sha(a) != rec["a_sha256"]:
            mism = int((a[::g["sample_stride"]] != asamp).sum()) if t == T else -1
            pytest.fail(f"{name} t={t}: assignments differ from the oracle's (sampled mismatches at T: {mism})")
        C = km.centroids()
        err = centroid_rel_err(C, Cg[t - 1]).max()
        assert err <= 1e-12, (t, err)
        st = km.stats()[-1]
        assert changed == rec["changed"] and st["empty"] == rec["empty"], (t, changed, rec)
        assert abs(dists - rec["dists"]) <= 1e-3 * rec["dists"], (t, dists, rec["dists"])
        assert abs(st["clause1"] - rec["clause1"]) <= 1e-3 * spec.n, (t, st["clause1"], rec["clause1"])
        sse = km.sse()
        assert abs(sse - rec["sse"]) <= 1e-12 * rec["sse"], (t, sse, rec["sse"])
        if t in check_at:
            _independent_checks(X, a, km.bounds(), Cused, rng, 200_000 if spec.k <= 100 else 40_000)
        if changed <= spec.tol:
            break
    assert t == T
    assert np.array_equal(a[::g["sample_stride"]], asamp)
    assert abs(km.sse() - g["final_sse"]) <= 1e-12 * g["final_sse"]
    # exact-order sums of a_T (reading B12) reproduce the oracle's C_T bit for bit
    km.finalize()
    assert np.array_equal(km.centroids(), Cg[T - 1]), float(np.abs(km.centroids() - Cg[T - 1]).max())
    assert abs(km.sse() - g["final_sse"]) <= 1e-12 * g["final_sse"]
    km.close()
