"""Synthetic data recipe ("Synthetic inputs"; BASELINE.json ``configs``).

The paper's datasets (Friendster-8/32 eigenvectors, RM/RU random sets; PAPER.md:236-261,
Table "datasets under evaluation") are not available, so these seeded generators stand in
for them with the same shapes, scales and structure:

* ``mixture``  — isotropic Gaussian mixtures (C1, C2, C5): stand-ins for the paper's
  "Rand-Multivariate" sets.
* ``spectral`` — heavy-tailed Student-t(3) columns normalised to unit L2 norm and scaled by
  1/(j+1) (C3, C4): stand-ins for the top-8/top-32 eigenvectors of Friendster
  (PAPER.md:141-150, 245-249).

Recipe (numpy PCG64; ``rng(*key) = default_rng(SeedSequence(seed, spawn_key=key))``; seed 0;
chunks of CH = 2**20 rows so the bytes do not depend on the worker count):

* mixture: ``p = rng(0,0)``: ``means = p.uniform(-R, R, (K, d))``; only for C2
  ``sig = p.uniform(0.5, 2.0, K)`` then ``w = p.dirichlet(ones(K))``.  Chunk c:
  ``lab = rng(1,c).choice(K, m, p=w)``, ``z = rng(2,c).standard_normal((m, d))``,
  ``X = fp32(means[lab] + sig[lab, None] * z)``.
* spectral: column j, chunk c: ``raw = rng(2,j,c).standard_t(3, m)``; ``ss_j`` = sum over
  chunks (in chunk order) of ``dot(raw, raw)``; ``X[:, j] = fp32((raw / sqrt(ss_j)) / (j+1))``.
  C3 = C4[:, :8].
* Forgy: ``idx = rng(3,0).choice(n, k, replace=False)`` (BASELINE.json: "k distinct points
  chosen by seeded uniform sampling").

Generation is parallelised over (column, chunk) tasks with a fork pool writing into a shared
anonymous mapping; the result is byte-identical to the serial recipe.
"""
from __future__ import annotations

import hashlib
import mmap
import os
from dataclasses import dataclass
from typing import Optional, Tuple

import numpy as np

CH = 1 << 20  # rows per chunk
RECIPE_VERSION = "survey-8d-v1"


@dataclass(frozen=True)
class ConfigSpec:
    name: str
    n: int
    d: int
    k: int
    kind: str          # "mixture" | "spectral"
    max_iters: int
    tol: int = 0       # stop iff changed <= tol (a count of points)
    K: int = 0         # mixture components
    R: float = 0.0     # mixture mean range [-R, R]
    sigma_range: Optional[Tuple[float, float]] = None  # per-component sigma ~ U[a, b] (C2)
    dirichlet: bool = False                             # mixture weights ~ Dirichlet(1) (C2)


CONFIGS = {
    "c1": ConfigSpec("c1", 10_000, 8, 10, "mixture", 100, K=10, R=10.0),
    "c2": ConfigSpec("c2", 1_000_000, 16, 100, "mixture", 50, K=100, R=20.0,
                     sigma_range=(0.5, 2.0), dirichlet=True),
    "c3": ConfigSpec("c3", 65_608_366, 8, 100, "spectral", 30),
    "c4": ConfigSpec("c4", 65_608_366, 32, 100, "spectral", 30),
    "c5": ConfigSpec("c5", 100_000_000, 32, 1000, "mixture", 20, K=1000, R=50.0),
}


def _rng(seed: int, *key: int) -> np.random.Generator:
    return np.random.default_rng(np.random.SeedSequence(seed, spawn_key=tuple(key)))


def _chunks(n: int):
    c = 0
    while c * CH < n:
        lo = c * CH
        yield c, lo, min(n, lo + CH)
        c += 1


# ----------------------------------------------------------------------------------------
# shared output buffer + fork pool plumbing
_SHARED = {}


def _shared_array(shape, dtype) -> np.ndarray:
    nbytes = int(np.prod(shape)) * np.dtype(dtype).itemsize
    buf = mmap.mmap(-1, max(nbytes, 1), flags=mmap.MAP_SHARED)
    arr = np.frombuffer(buf, dtype=dtype, count=int(np.prod(shape))).reshape(shape)
    return arr


def _workers(workers: Optional[int]) -> int:
    if workers is not None:
        return max(1, workers)
    env = os.environ.get("SYNTH_WORKERS")
    if env:
        return max(1, int(env))
    return max(1, min(32, os.cpu_count() or 1))


def _pool_map(fn, tasks, workers: int):
    if workers <= 1 or len(tasks) <= 1:
        return [fn(t) for t in tasks]
    import multiprocessing as mp
    ctx = mp.get_context("fork")
    with ctx.Pool(min(workers, len(tasks))) as pool:
        return pool.map(fn, tasks, chunksize=1)


# ---- mixture ----------------------------------------------------------------------------
def _mixture_params(spec: ConfigSpec, d: int, seed: int):
    p = _rng(seed, 0, 0)
    means = p.uniform(-spec.R, spec.R, (spec.K, d))
    if spec.sigma_range is not None:
        sig = p.uniform(spec.sigma_range[0], spec.sigma_range[1], spec.K)
    else:
        sig = np.ones(spec.K)
    if spec.dirichlet:
        w = p.dirichlet(np.ones(spec.K))
    else:
        w = np.full(spec.K, 1.0 / spec.K)
    return means, sig, w


def _mixture_task(args):
    c, lo, hi = args
    st = _SHARED["mix"]
    means, sig, w, seed, out = st["means"], st["sig"], st["w"], st["seed"], st["out"]
    m = hi - lo
    lab = _rng(seed, 1, c).choice(len(w), m, p=w)
    z = _rng(seed, 2, c).standard_normal((m, means.shape[1]))
    out[lo:hi] = (means[lab] + sig[lab, None] * z).astype(np.float32)
    return None


def _mixture_task_rows(args):
    c, lo, hi, rlo, rhi = args
    st = _SHARED["mix"]
    means, sig, w, seed, out = st["means"], st["sig"], st["w"], st["seed"], st["out"]
    m = hi - lo
    lab = _rng(seed, 1, c).choice(len(w), m, p=w)
    z = _rng(seed, 2, c).standard_normal((m, means.shape[1]))
    a, b = max(lo, rlo), min(hi, rhi)
    out[a - rlo:b - rlo] = (means[lab[a - lo:b - lo]] + sig[lab[a - lo:b - lo], None]
                            * z[a - lo:b - lo]).astype(np.float32)
    return None


def _make_mixture(spec: ConfigSpec, n: int, seed: int, workers: int, rows=None) -> np.ndarray:
    means, sig, w = _mixture_params(spec, spec.d, seed)
    rlo, rhi = (0, n) if rows is None else rows
    out = _shared_array((rhi - rlo, spec.d), np.float32)
    _SHARED["mix"] = dict(means=means, sig=sig, w=w, seed=seed, out=out)
    try:
        if rows is None:
            _pool_map(_mixture_task, list(_chunks(n)), workers)
        else:
            tasks = [(c, lo, hi, rlo, rhi) for (c, lo, hi) in _chunks(n) if hi > rlo and lo < rhi]
            _pool_map(_mixture_task_rows, tasks, workers)
    finally:
        _SHARED.pop("mix", None)
    return out


# ---- spectral ---------------------------------------------------------------------------
def _spectral_dot_task(args):
    j, c, lo, hi, seed = args
    raw = _rng(seed, 2, j, c).standard_t(3, hi - lo)
    return float(np.dot(raw, raw))


def _spectral_fill_task(args):
    j, c, lo, hi, seed = args
    st = _SHARED["spec"]
    rlo, rhi = st["rows"]
    a, b = max(lo, rlo), min(hi, rhi)
    raw = _rng(seed, 2, j, c).standard_t(3, hi - lo)[a - lo:b - lo]
    st["out"][a - rlo:b - rlo, j] = ((raw / st["norm"][j]) / (j + 1)).astype(np.float32)
    return None


def _make_spectral(spec: ConfigSpec, n: int, d: int, seed: int, workers: int, rows=None) -> np.ndarray:
    chunks = list(_chunks(n))
    tasks = [(j, c, lo, hi, seed) for j in range(d) for (c, lo, hi) in chunks]
    dots = _pool_map(_spectral_dot_task, tasks, workers)   # column norms need every row
    nch = len(chunks)
    norm = np.empty(d)
    for j in range(d):
        ss = 0.0
        for c in range(nch):          # fp64, chunk order
            ss += dots[j * nch + c]
        norm[j] = np.sqrt(ss)
    rlo, rhi = (0, n) if rows is None else rows
    out = _shared_array((rhi - rlo, d), np.float32)
    _SHARED["spec"] = dict(out=out, norm=norm, rows=(rlo, rhi))
    try:
        _pool_map(_spectral_fill_task, [t for t in tasks if t[3] > rlo and t[2] < rhi], workers)
    finally:
        _SHARED.pop("spec", None)
    return out


# ---- public -----------------------------------------------------------------------------
def make_points(name: str, n: Optional[int] = None, seed: int = 0,
                workers: Optional[int] = None, rows: Optional[Tuple[int, int]] = None) -> np.ndarray:
    """X (n x d, fp32, C-contiguous) for config ``name``.  ``n`` overrides the row count
    (a smaller instance of the same recipe, used for parity cases; for ``spectral`` a
    smaller n changes the column norms, so it is a new instance of the same distribution,
    not a prefix).  ``rows=(lo, hi)`` returns only those rows of the n-row matrix (a rank's
    shard), byte-identical to slicing the full matrix."""
    spec = CONFIGS[name]
    n = spec.n if n is None else int(n)
    w = _workers(workers)
    if rows is not None:
        rows = (int(rows[0]), int(rows[1]))
        assert 0 <= rows[0] <= rows[1] <= n
    if spec.kind == "mixture":
        return _make_mixture(spec, n, seed, w, rows)
    return _make_spectral(spec, n, spec.d, seed, w, rows)


def forgy_indices(n: int, k: int, seed: int = 0) -> np.ndarray:
    """k distinct row indices, drawn without replacement (SURVEY.md §8(d) "Forgy")."""
    if k > n:
        raise ValueError("k > n")
    return _rng(seed, 3, 0).choice(n, k, replace=False).astype(np.int64)


def sha256_points(X: np.ndarray) -> str:
    h = hashlib.sha256()
    flat = np.ascontiguousarray(X, dtype=np.float32).reshape(-1)
    step = 1 << 26
    for i in range(0, flat.size, step):
        h.update(flat[i:i + step].tobytes())
    return h.hexdigest()


def make_config(name: str, n: Optional[int] = None, seed: int = 0,
                workers: Optional[int] = None):
    """(X fp32 n x d, forgy idx int64[k], manifest dict)."""
    spec = CONFIGS[name]
    X = make_points(name, n=n, seed=seed, workers=workers)
    idx = forgy_indices(X.shape[0], spec.k, seed)
    manifest = dict(config=name, n=int(X.shape[0]), d=spec.d, k=spec.k, seed=seed,
                    recipe=RECIPE_VERSION, numpy=np.__version__, idx_head=idx[:8].tolist())
    return X, idx, manifest
