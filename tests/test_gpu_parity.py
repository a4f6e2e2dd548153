"""GPU parity: the CUDA path (through the C ABI) against the fp64 CPU oracle.

Strict tier (exact mode): free-running assignments identical to the oracle's at
every iteration, centroids <= 1e-12 relative, SSE <= 1e-12 relative, equal iteration counts.
BASELINE tier (the contract): outside the near-tie set assignments bit-exact; centroids
<= 1e-5; SSE <= 1e-4.  We assert the strict tier where it is the expected outcome.
"""
import json
import os

import numpy as np
import pytest

import oracle
from helpers import centroid_rel_err, near_tie_mask
from synth import CONFIGS, make_config

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1902_09527_b200 import KMeans, KMeansError  # noqa: E402

HV = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "hand_vectors.json")))


def gpu_run(X, C0, max_iters, prune="mti", tol=0, **kw):
    Xd = torch.from_numpy(np.ascontiguousarray(X, np.float32)).cuda()
    km = KMeans(Xd, C0, prune=prune, **kw)
    it, dists = km.run(max_iters, tol)
    out = dict(iterations=it, dists=dists, a=km.assignments(), C=km.centroids(), sse=km.sse(),
               stats=km.stats(), launches=km.launch_count)
    km.close()
    return out


def assert_strict(g, r, exact_C=True):
    """exact_C: kmeans_run ends with kmeans_finalize, whose sums follow the oracle's order
    (reading B12: 64 Ki-row blocks in row order, merged in block order), so with equal
    assignments the centroids are bit-identical to the oracle's."""
    assert g["iterations"] == r.iterations
    assert np.array_equal(g["a"], r.a), int((g["a"] != r.a).sum())
    assert centroid_rel_err(g["C"], r.C).max() <= 1e-12
    if exact_C:
        assert np.array_equal(g["C"], r.C), float(np.abs(g["C"] - r.C).max())
    assert abs(g["sse"] - r.final_sse) <= 1e-12 * max(r.final_sse, 1e-300) + 1e-300
    assert [s["changed"] for s in g["stats"]] == r.changed.tolist()
    assert [s["empty"] for s in g["stats"]] == r.empty.tolist()


# ---- hand-checked vectors ------------------------------------------------------------------
@pytest.mark.parametrize("prune", ["mti", "none"])
def test_B1(prune):
    e = HV["B1"]
    g = gpu_run(np.array(e["X"], np.float32), np.array(e["C0"], float), 100, prune)
    assert g["iterations"] == 2 and g["a"].tolist() == e["a_T"]
    assert np.array_equal(g["C"], np.array(e["C_T"], float)) and g["sse"] == e["sse"]
    assert [s["dists"] for s in g["stats"]] == e[("mti" if prune == "mti" else "brute") + "_dists"]


def test_B2_trace():
    e = HV["B2"]
    X = np.array(e["X"], np.float32)
    g = gpu_run(X, X[e["forgy"]].astype(float), 100, "mti")
    assert g["iterations"] == e["iterations"]
    assert [s["dists"] for s in g["stats"]] == e["dists"]
    assert [s["changed"] for s in g["stats"]] == e["changed"]
    assert [s["clause1"] for s in g["stats"]] == e["clause1"]
    assert np.allclose(g["C"], np.array(e["C_T"], float), atol=1e-12, rtol=0)
    assert abs(g["sse"] - e["sse"]) < 1e-9


@pytest.mark.parametrize("prune", ["mti", "none"])
def test_B5_empty_cluster(prune):
    e = HV["B5"]
    X = np.array(e["X"], np.float32)
    g = gpu_run(X, X[e["forgy"]].astype(float), 100, prune)
    assert g["iterations"] == e["iterations"] and g["a"].tolist() == e["a_T"]
    assert np.allclose(g["C"], np.array(e["C_T"], float), atol=1e-12, rtol=0)
    assert [s["empty"] for s in g["stats"]] == e["empty"]
    assert abs(g["sse"] - e["sse"]) < 1e-12


def test_B3_half_factor_on_gpu():
    """x=(1.5,0) between (0,0) and (2,0): must end in cluster 1 (the literal clause would not)."""
    X = np.array([[1.5, 0.0], [0.0, 0.0], [2.0, 0.0], [-3.0, 0.0], [5.0, 0.0]], np.float32)
    C0 = np.array([[0.0, 0.0], [2.0, 0.0]])
    r = oracle.lloyd(X, C0, 50, 0, "brute")
    assert_strict(gpu_run(X, C0, 50, "mti"), r)


# ---- seeded configs, free-running (strict tier) -------------------------------------------
@pytest.mark.parametrize("prune,engine", [("mti", "tensor"), ("mti", "cuda"), ("mti", "screen"), ("mti", "tensor_screen"), ("mti", "tensor_chunked"), ("none", "auto")])
def test_c1_free_running(prune, engine):
    X, idx, _ = make_config("c1")
    C0 = X[idx].astype(float)
    r = oracle.lloyd(X, C0, 100, 0, "mti")
    g = gpu_run(X, C0, 100, prune, engine=engine)
    assert_strict(g, r)
    if prune == "mti":
        # distance counts vs oracle-mti: soft 0.1 % (fp32 vs fp64 bound rounding)
        gd = np.array([s["dists"] for s in g["stats"]])
        assert np.all(np.abs(gd - r.dists) <= 1e-3 * r.dists + 1)
        gc = np.array([s["clause1"] for s in g["stats"]])
        assert np.all(np.abs(gc - r.clause1) <= 1e-3 * 10000 + 1)


@pytest.mark.parametrize("prune,engine", [("mti", "tensor"), ("mti", "cuda"), ("mti", "screen"), ("mti", "tensor_screen"), ("mti", "tensor_chunked"), ("none", "auto")])
def test_c2_free_running(prune, engine):
    X, idx, _ = make_config("c2")
    C0 = X[idx].astype(float)
    r = oracle.lloyd(X, C0, 50, 0, "mti")
    g = gpu_run(X, C0, 50, prune, engine=engine)
    assert_strict(g, r)
    if prune == "mti":
        gd = np.array([s["dists"] for s in g["stats"]])
        assert np.all(np.abs(gd - r.dists) <= 1e-3 * r.dists)


@pytest.mark.parametrize("engine", ["tensor", "cuda", "screen", "tensor_screen", "tensor_chunked"])
@pytest.mark.parametrize("name,n,iters", [("c3", 2_000_000, 30), ("c4", 1_000_000, 30)])
def test_spectral_shaped_free_running(name, n, iters, engine):
    X, idx, _ = make_config(name, n=n)
    C0 = X[idx].astype(float)
    r = oracle.lloyd(X, C0, iters, 0, "mti")
    g = gpu_run(X, C0, iters, "mti", engine=engine)
    assert_strict(g, r)
    gd = np.array([s["dists"] for s in g["stats"]])
    assert np.all(np.abs(gd - r.dists) <= 1e-3 * r.dists)


@pytest.mark.parametrize("engine", ["tensor", "cuda", "screen", "tensor_screen", "tensor_chunked"])
def test_c5_shaped_large_k(engine):
    X, idx, _ = make_config("c5", n=300_000)
    C0 = X[idx].astype(float)
    r = oracle.lloyd(X, C0, 8, 0, "mti")
    g = gpu_run(X, C0, 8, "mti", engine=engine)
    assert_strict(g, r)


# ---- lockstep, BASELINE tier with near-tie exclusion ---------------------------------------
def test_c2_lockstep_single_step():
    X, idx, _ = make_config("c2")
    C0 = X[idx].astype(float)
    Xd = torch.from_numpy(X).cuda()
    km = KMeans(Xd, C0, prune="mti")
    Cprev = C0
    for t in range(1, 8):
        # oracle single step from the same centroids
        a_o, d1, d2 = oracle.assign_brute(X, Cprev)
        km.set_centroids(Cprev)
        km.iterate()
        a_g = km.assignments()
        ties = near_tie_mask(d1, d2)
        assert np.array_equal(a_g[~ties], a_o[~ties])
        assert np.array_equal(a_g, a_o)          # exact mode: no exclusions needed
        sums, counts = oracle.cluster_sums(X, a_g, 100)
        C_from_gpu_a, _ = oracle.update(sums, counts, Cprev)
        Cg = km.centroids()
        assert centroid_rel_err(Cg, C_from_gpu_a).max() <= 1e-12
        Cprev = Cg
    km.close()


# ---- edge cases ------------------------------------------------------------------------------
@pytest.mark.parametrize("engine", ["cuda", "screen"])
@pytest.mark.parametrize("d", [1, 2, 3, 5, 12, 20, 32, 33, 64])
def test_dims_padding(d, engine):
    rng = np.random.default_rng(d)
    X = (rng.normal(size=(3001, d)) + rng.integers(0, 4, size=(3001, 1)) * 3).astype(np.float32)
    C0 = X[rng.choice(3001, 7, replace=False)].astype(float)
    r = oracle.lloyd(X, C0, 60, 0, "brute")
    for prune in ("mti", "none"):
        assert_strict(gpu_run(X, C0, 60, prune, engine=engine), r)


@pytest.mark.parametrize("k", [2, 7, 23, 24, 25, 26, 40, 112])
def test_walk_table_head_boundaries(k):
    """d = 32 walk with the per-warp shared-memory copy of the first 24 candidates of the warp
    cluster's list (km_walk_common.cuh, walk_tab_cap): lists shorter than, equal to and longer than
    the copied head (the tail is read from global memory), overlapping clusters so that walks are
    long and rows move between clusters for many iterations."""
    rng = np.random.default_rng(1000 + k)
    n = 40_003
    means = rng.uniform(-3, 3, size=(k, 32))
    X = (means[rng.integers(0, k, size=n)] + rng.normal(size=(n, 32)) * 2.0).astype(np.float32)
    C0 = X[rng.choice(n, k, replace=False)].astype(float)
    r = oracle.lloyd(X, C0, 25, 0, "brute")
    assert_strict(gpu_run(X, C0, 25, "mti", engine="cuda"), r)


@pytest.mark.parametrize("engine", ["cuda", "screen", "tensor_screen", "tensor_chunked"])
@pytest.mark.parametrize("n", [1, 5, 31, 33, 257, 1000])
def test_small_and_ragged_n(n, engine):
    rng = np.random.default_rng(n)
    X = rng.normal(size=(n, 8 if engine.startswith("tensor") else 4)).astype(np.float32)   # tcgen05: d padded to 8/16/32
    k = min(n, 3)
    C0 = X[:k].astype(float)
    r = oracle.lloyd(X, C0, 30, 0, "brute")
    assert_strict(gpu_run(X, C0, 30, "mti", engine=engine), r)


def test_k1_and_k_equals_n():
    rng = np.random.default_rng(3)
    X = rng.normal(size=(500, 3)).astype(np.float32)
    r = oracle.lloyd(X, X[:1].astype(float), 10, 0, "mti")
    g = gpu_run(X, X[:1].astype(float), 10, "mti")
    assert_strict(g, r)
    assert [s["dists"] for s in g["stats"]] == [500, 0]
    Xs = X[:40]
    r = oracle.lloyd(Xs, Xs.astype(float), 10, 0, "brute")
    g = gpu_run(Xs, Xs.astype(float), 10, "mti")
    assert_strict(g, r)
    assert g["sse"] == 0.0


@pytest.mark.parametrize("engine", ["cuda", "screen", "tensor_screen", "tensor_chunked"])
@pytest.mark.parametrize("policy", ["never", "always", "auto"])
def test_resort_policies_agree(policy, engine):
    X, idx, _ = make_config("c3", n=400_000)
    C0 = X[idx].astype(float)
    r = oracle.lloyd(X, C0, 12, 0, "mti")
    assert_strict(gpu_run(X, C0, 12, "mti", resort=policy, engine=engine), r)


def test_max_iters_zero_and_host_points():
    X, idx, _ = make_config("c1")
    C0 = X[idx].astype(float)
    km = KMeans(X, C0)                        # host points: library copies H2D
    assert km.run(0, 0) == (0, 0)
    assert np.array_equal(km.centroids(), C0)
    with pytest.raises(KMeansError):
        km.assignments()                      # KM_ESTATE before iteration 1
    it, _ = km.run(100, 0)
    r = oracle.lloyd(X, C0, 100, 0, "brute")
    assert it == r.iterations and np.array_equal(km.assignments(), r.a)
    out = torch.empty(X.shape[0], dtype=torch.int32, device="cuda")
    km.assignments(out=out)
    assert np.array_equal(out.cpu().numpy(), r.a)
    km.close()


def test_usage_errors():
    X = np.zeros((4, 2), np.float32)
    with pytest.raises(KMeansError, match="KM_EARG"):
        KMeans(X, np.zeros((5, 2)))           # k > n
    with pytest.raises(KMeansError, match="KM_EARG"):
        KMeans(np.zeros((4, 65), np.float32), np.zeros((2, 65)))
    Xn = np.ones((10, 2), np.float32)
    Xn[3, 1] = np.nan
    with pytest.raises(KMeansError, match="KM_ENONFINITE"):
        KMeans(Xn, np.zeros((2, 2)), check_finite=True)
    with pytest.raises(KMeansError, match="KM_ENONFINITE"):
        KMeans(np.ones((10, 2), np.float32), np.array([[0, np.inf], [1, 1]]), check_finite=True)


@pytest.mark.parametrize("engine", ["cuda", "screen", "tensor_screen", "tensor_chunked"])
def test_bound_soundness_sampled(engine):
    """u_i >= ||x_i - C_used[a_i]|| (fp64, against the fp64 centroids the pass used) for every row
    after every pass, read through kmeans_get_bounds (u loosened by drift,
    tightened by U(u)); assignments equal the fp64 brute-force argmin of C_used."""
    X, idx, _ = make_config("c2")
    C0 = X[idx].astype(float)
    Xd = torch.from_numpy(X).cuda()
    km = KMeans(Xd, C0, prune="mti", engine=engine)
    with pytest.raises(KMeansError, match="KM_ESTATE"):
        km.bounds()
    for _ in range(8):
        Cused = km.centroids()
        km.iterate()
        a = km.assignments()
        u = km.bounds().astype(np.float64)
        a_o, d1, _ = oracle.assign_brute(X, Cused)
        assert np.array_equal(a, a_o)
        assert np.all(u >= np.sqrt(d1) * (1 - 1e-14)), int((u < np.sqrt(d1)).sum())
    km.close()


# ---- spherical k-means (§4.2) -------------------
@pytest.mark.parametrize("cfg,n", [("c1", None), ("c2", None), ("c3", 1_000_000)])
def test_skmeans_free_running(cfg, n):
    """sk-means through the same MTI engine: rows and centroids on the unit sphere (exact-mode
    arithmetic of the normalisation matches the oracle's step for step); strict parity."""
    X, idx, spec = make_config(cfg, n=n)
    C0 = X[idx].astype(float)
    iters = 30 if cfg != "c1" else 100
    r = oracle.skmeans(X, C0, iters, 0)
    g = gpu_run(X, C0, iters, "mti", spherical=True)
    assert g["iterations"] == r.iterations
    assert np.array_equal(g["a"], r.a), int((g["a"] != r.a).sum())
    assert centroid_rel_err(g["C"], r.C).max() <= 1e-12
    assert np.allclose(np.linalg.norm(g["C"], axis=1), 1.0, rtol=0, atol=1e-12)
    assert [s["changed"] for s in g["stats"]] == r.changed.tolist()
    assert abs(g["sse"] - r.final_sse) <= 1e-10 * r.final_sse


def test_skmeans_zero_row_rejected():
    X = np.array([[1, 0], [0, 0], [0, 2]], np.float32)
    Xd = torch.from_numpy(X).cuda()
    with pytest.raises(KMeansError):
        KMeans(Xd, X[[0, 2]].astype(float), spherical=True)


# ---- k-means++ D² seeding (Eq. 2) ---------------------------------
@pytest.mark.parametrize("cfg,n", [("c1", None), ("c2", 200_000), ("c3", 300_000)])
def test_seed_plusplus_matches_oracle(cfg, n):
    """The GPU draws the same rows as the oracle for the same uniforms (reading B9: the first row
    whose exact prefix sum of D² exceeds u times the exact total), from device and from host
    memory; the seeded run then matches the oracle's Lloyd from those centroids."""
    from paper_1902_09527_b200 import seed_plusplus
    X, _, spec = make_config(cfg, n=n)
    k = spec["k"]
    rng = np.random.default_rng(17)
    u = rng.random(k - 1)
    first = int(rng.integers(X.shape[0]))
    ch_o, C_o = oracle.seed_plusplus(X, k, u, first)
    ch_g, C_g = seed_plusplus(torch.from_numpy(X).cuda(), k, u, first)
    assert ch_g.tolist() == ch_o.tolist()
    assert np.array_equal(C_g, C_o)
    ch_h, _ = seed_plusplus(X, k, u, first)
    assert ch_h.tolist() == ch_o.tolist()
    if cfg == "c1":
        r = oracle.lloyd(X, C_o, 100, 0, "mti")
        assert_strict(gpu_run(X, C_g, 100), r)


def test_seed_plusplus_exact_crossing():
    """D² = (0, 2^53, 1, 1) from fp32 rows (0,0), (2^26,2^26), (1,0), (0,1), first row 0, u the
    largest double below 1: the exact target 2^53 + 1 - 2^-52 is first exceeded at row 2 (fp64
    running sums, which round 2^53 + 1 to 2^53, would give row 1 or 3)."""
    from paper_1902_09527_b200 import seed_plusplus
    X = np.array([[0, 0], [2.0 ** 26, 2.0 ** 26], [1, 0], [0, 1]], np.float32)
    u = [float(np.nextafter(1.0, 0.0))]
    ch_o, _ = oracle.seed_plusplus(X, 2, u, 0)
    ch_g, _ = seed_plusplus(torch.from_numpy(X).cuda(), 2, u, 0)
    assert ch_o.tolist() == [0, 2] and ch_g.tolist() == [0, 2]
    # the same at scale: 3 M rows of unit weight behind one row of weight 2^53
    n = 3_000_000
    Xb = np.zeros((n, 2), np.float32)
    Xb[1] = 2.0 ** 26
    Xb[2:, 0] = 1.0
    ch_g, _ = seed_plusplus(torch.from_numpy(Xb).cuda(), 2, u, 0)
    # exact: total T = 2^53 + n - 2, u T = 2^53 + n - 3 - (n - 2) 2^-53; the prefix through row
    # i >= 1 is 2^53 + i - 1, first above u T at i = n - 2
    assert ch_g.tolist() == [0, n - 2]


def test_seed_plusplus_errors():
    from paper_1902_09527_b200 import seed_plusplus
    X = np.ones((4, 3), np.float32)
    with pytest.raises(KMeansError):
        seed_plusplus(X, 2, [0.5], 0)            # fewer than k distinct rows
    with pytest.raises(KMeansError):
        seed_plusplus(np.eye(3, dtype=np.float32), 2, [1.5], 0)


def test_kmeanspp_multirun_matches_oracle():
    """k-means++ with r = 3 runs on C1: same best run, assignments and centroids as the oracle."""
    from paper_1902_09527_b200 import kmeanspp_multirun
    X, _, spec = make_config("c1")
    rng = np.random.default_rng(23)
    runs = [(int(rng.integers(X.shape[0])), rng.random(spec["k"] - 1)) for _ in range(3)]
    bo = oracle.kmeanspp_multirun(X, spec["k"], runs, 100)
    bg = kmeanspp_multirun(torch.from_numpy(X).cuda(), spec["k"], runs, 100)
    assert bg[0] == bo[0] and bg[4] == bo[4]
    assert np.array_equal(bg[1], bo[1])
    assert centroid_rel_err(bg[2], bo[2]).max() <= 1e-12
    assert abs(bg[3] - bo[3]) <= 1e-12 * bo[3]


@pytest.mark.parametrize("d,k", [(3, 1), (5, 7), (33, 4)])
def test_skmeans_and_seed_odd_shapes(d, k):
    """sk-means and k-means++ seeding with padded row widths (d -> DP) and k = 1."""
    from paper_1902_09527_b200 import seed_plusplus
    rng = np.random.default_rng(d * 100 + k)
    X = (rng.normal(size=(5000, d)) + rng.normal(size=(1, d)) * 3).astype(np.float32)
    u = rng.random(max(k - 1, 0))
    ch_o, C_o = oracle.seed_plusplus(X, k, u, 17)
    ch_g, C_g = seed_plusplus(X, k, u, 17)
    assert ch_g.tolist() == ch_o.tolist() and np.array_equal(C_g, C_o)
    r = oracle.skmeans(X, C_o, 50, 0)
    g = gpu_run(X, C_g, 50, "mti", spherical=True)
    assert g["iterations"] == r.iterations and np.array_equal(g["a"], r.a)
    assert centroid_rel_err(g["C"], r.C).max() <= 1e-12


# ---- CUDA graph replay and the collective path ------------------------------------
def test_graph_replay_equals_eager():
    """Iterations t >= 2 replayed from a captured CUDA graph (default) give the same assignments,
    centroids and per-iteration counts as eager launches, across re-bucketing (both row buffers)."""
    X, idx, _ = make_config("c3", n=400_000)
    C0 = X[idx].astype(float)
    g = gpu_run(X, C0, 20, "mti")
    e = gpu_run(X, C0, 20, "mti", graph=False)
    assert g["iterations"] == e["iterations"] and np.array_equal(g["a"], e["a"])
    assert np.array_equal(g["C"], e["C"])
    for f in ("changed", "dists", "clause1", "empty", "resorted"):
        assert [s[f] for s in g["stats"]] == [s[f] for s in e["stats"]], f
    assert sum(s["resorted"] for s in g["stats"][1:]) >= 1


def test_nccl_path_at_world_1():
    """The library's NCCL data path (communicator from a fresh ncclUniqueId, one allreduce of
    [sums | counts] and the counters per iteration, captured in the iteration graph; SSE
    allreduce) on a 1-rank communicator: strict parity with the oracle."""
    from paper_1902_09527_b200 import nccl_unique_id
    X, idx, _ = make_config("c2")
    C0 = X[idx].astype(float)
    r = oracle.lloyd(X, C0, 50, 0, "mti")
    for graph in (True, False):
        g = gpu_run(X, C0, 50, "mti", nccl_id=nccl_unique_id(), force_comm=True, graph=graph)
        assert_strict(g, r)
        assert all(s["ms_comm"] > 0 for s in g["stats"])


def _two_gpu_worker(rank, port, X, C0, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=2)
    from paper_1902_09527_b200 import KMeans as KM, nccl_unique_id
    from paper_1902_09527_b200.dist import broadcast_bytes, shard_bounds
    lo, hi = shard_bounds(X.shape[0], rank, 2)
    nid = broadcast_bytes(nccl_unique_id() if rank == 0 else b"\0" * 128)
    km = KM(torch.from_numpy(X[lo:hi]).cuda(), C0, rank=rank, world=2, nccl_id=nid, n_global=X.shape[0])
    it, _ = km.run(50, 0)
    q.put((rank, it, km.assignments(), km.centroids(), km.sse()))
    km.close()
    dist.destroy_process_group()


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_two_gpus_equal_one():
    """G = 2 contiguous shards (§7) vs G = 1: same iterations and assignments, centroids
    bitwise identical on both ranks and <= 1e-12 from G = 1 (only the fp64 reduction order differs)."""
    import socket
    import torch.multiprocessing as mp
    X, idx, _ = make_config("c2")
    C0 = X[idx].astype(float)
    one = gpu_run(X, C0, 50, "mti")
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_two_gpu_worker, args=(r, port, X, C0, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=600) for _ in range(2))
    for p in ps:
        p.join(timeout=60)
    (_, it0, a0, Ca, s0), (_, it1, a1, Cb, s1) = res
    assert it0 == it1 == one["iterations"]
    assert np.array_equal(np.concatenate([a0, a1]), one["a"])
    assert np.array_equal(Ca, Cb) and centroid_rel_err(Ca, one["C"]).max() <= 1e-12
    assert s0 == s1 and abs(s0 - one["sse"]) <= 1e-12 * one["sse"]


def test_periodic_full_resummation():
    """Running sums updated by deltas (reading B5) are re-derived from every row once the moves
    since the last full reduction exceed resum_moves * n: with a tiny threshold (a full
    reduction almost every iteration) the run is still strict-parity with the oracle."""
    X, idx, _ = make_config("c2")
    C0 = X[idx].astype(float)
    r = oracle.lloyd(X, C0, 50, 0, "mti")
    assert_strict(gpu_run(X, C0, 50, "mti", resum_moves=0.01), r)


def test_long_run_delta_sums_do_not_drift():
    """200 iterations of C2 with delta sums only (no re-summation): the centroids stay within
    1e-12 of the oracle's means of the GPU's own assignments (fp64 rounding of ~1e6 moves);
    kmeans_finalize then re-derives them in the oracle's order: bit-identical."""
    X, idx, _ = make_config("c2")
    C0 = X[idx].astype(float)
    Xd = torch.from_numpy(X).cuda()
    km = KMeans(Xd, C0, prune="mti", resum_moves=-1.0)
    for _ in range(200):
        if km.iterate()[0] == 0:
            break
    a = km.assignments()
    C_run = km.centroids()
    sums, counts = oracle.cluster_sums(X, a, 100)
    prev = km.stats()
    moved = sum(s["changed"] for s in prev[1:])
    assert moved > 0
    # the update of the last pass: empty clusters keep the centroids that pass used
    C_means, _ = oracle.update(sums, counts, C_run)
    assert centroid_rel_err(C_run, C_means).max() <= 1e-12
    km.finalize()
    assert np.array_equal(km.centroids(), C_means)
    km.close()


def test_finalize_is_bit_reproducible():
    """Two runs of C2 (delta sums applied in a timing-dependent order) end with bit-identical
    centroids after kmeans_finalize (reading B12), equal to the oracle's."""
    X, idx, _ = make_config("c2")
    C0 = X[idx].astype(float)
    g1 = gpu_run(X, C0, 50, "mti")
    g2 = gpu_run(X, C0, 50, "mti")
    assert np.array_equal(g1["a"], g2["a"]) and np.array_equal(g1["C"], g2["C"])
    r = oracle.lloyd(X, C0, 50, 0, "mti")
    assert np.array_equal(g1["C"], r.C)
