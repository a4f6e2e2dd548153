"""Python face of the C ABI: ``KMeans`` wraps one ``km_ctx`` (one rank's shard).

PyTorch is used only for device memory, streams and process groups; all arithmetic runs in
``libkmeans_b200.so``.  Method: Lloyd's k-means (§4.1, 1104-1130) with MTI pruning
(§3.3, 1013-1053); see include/kmeans_b200.h for the contract of each call.
"""
from __future__ import annotations

import ctypes as ct
from typing import Optional

import numpy as np

from . import _capi as C


def default_options() -> C.KmOptions:
    o = C.KmOptions()
    C.lib().kmeans_default_options(ct.byref(o))
    return o


def nccl_unique_id() -> bytes:
    buf = (ct.c_uint8 * 128)()
    C.check(C.lib().kmeans_nccl_unique_id(buf))
    return bytes(buf)


class KMeans:
    """One rank's k-means context.

    points: a contiguous fp32 (n_local x d) torch CUDA tensor (borrowed during construction)
            or a host array (numpy / CPU tensor; copied host->device by the library).
    init_centroids: (k x d) array, converted to fp64 on the host (copied).
    """

    def __init__(self, points, init_centroids, *, prune: str = "mti", device: Optional[int] = None,
                 stream=None, rank: int = 0, world: int = 1, nccl_id: Optional[bytes] = None,
                 n_global: int = 0, check_finite: bool = False, resort: str = "auto",
                 resort_fraction: float = 0.0, engine: str = "auto", spherical: bool = False,
                 graph: bool = True, force_comm: bool = False, resum_moves: float = 0.0):
        L = C.lib()
        o = default_options()
        self._keep = []
        on_host = True
        try:
            import torch
            if isinstance(points, torch.Tensor):
                if points.dtype != torch.float32 or not points.is_contiguous():
                    raise ValueError("points must be a contiguous float32 tensor")
                if points.is_cuda:
                    on_host = False
                    ptr = points.data_ptr()
                    dev = points.device.index if device is None else device
                    o.device = dev
                    if stream is None:
                        stream = torch.cuda.current_stream(dev).cuda_stream
                else:
                    points = points.numpy()
        except ImportError:
            pass
        if on_host:
            points = np.ascontiguousarray(points, dtype=np.float32)
            self._keep.append(points)
            ptr = points.ctypes.data
            o.device = 0 if device is None else device
        n, d = points.shape
        C0 = np.ascontiguousarray(init_centroids, dtype=np.float64).reshape(-1, d)
        self._keep.append(C0)
        if stream is not None:
            o.stream = ct.c_void_p(int(stream))
        o.prune = {"mti": C.KM_PRUNE_MTI, "none": C.KM_PRUNE_NONE, "ti": C.KM_PRUNE_TI}[prune]
        o.rank, o.world, o.n_global = rank, world, n_global
        if nccl_id is not None:
            o.nccl_unique_id[:] = list(nccl_id)
        o.check_finite = int(check_finite)
        o.points_on_host = int(on_host)
        o.resort_policy = {"auto": C.KM_RESORT_AUTO, "never": C.KM_RESORT_NEVER,
                           "always": C.KM_RESORT_ALWAYS}[resort]
        o.resort_fraction = resort_fraction
        o.engine = {"auto": C.KM_ENGINE_AUTO, "cuda": C.KM_ENGINE_CUDA_CORE,
                    "tensor": C.KM_ENGINE_TENSOR, "screen": C.KM_ENGINE_SCREEN,
                    "tensor_screen": C.KM_ENGINE_TENSOR_SCREEN, "tensor_chunked": C.KM_ENGINE_TENSOR_CHUNKED}[engine]
        o.spherical = int(bool(spherical))
        o.no_graph = int(not graph)
        o.force_comm = int(bool(force_comm))
        o.resum_moves = float(resum_moves)
        h = ct.c_void_p()
        C.check(L.kmeans_create(n, d, C0.shape[0], ptr, C0.ctypes.data, ct.byref(o), ct.byref(h)))
        self._h = h
        self._keep.clear()
        self.n, self.d, self.k = n, d, C0.shape[0]

    # -- one iteration / a run ----------------------------------------------------------------
    def iterate(self):
        ch, ds = ct.c_int64(), ct.c_int64()
        C.check(C.lib().kmeans_iterate(self._h, ct.byref(ch), ct.byref(ds)))
        return ch.value, ds.value

    def finalize(self):
        """C_T re-derived from exact-order sums of the current assignment (``kmeans_finalize``,
        DESIGN.md reading B12): bit-reproducible centroids.  ``run`` calls it."""
        C.check(C.lib().kmeans_finalize(self._h))

    def run(self, max_iters: int, tol: int = 0):
        it, ds = ct.c_int32(), ct.c_int64()
        C.check(C.lib().kmeans_run(self._h, int(max_iters), int(tol), ct.byref(it), ct.byref(ds)))
        return it.value, ds.value

    # -- results -------------------------------------------------------------------------------
    def assignments(self, out=None):
        """int32[n_local] in the caller's row order.  ``out`` may be an int32 torch tensor on the
        context's device or in (preferably pinned) host memory, or an int32 numpy array."""
        if out is not None:
            if hasattr(out, "data_ptr"):
                on_dev = 1 if getattr(out, "is_cuda", False) else 0
                C.check(C.lib().kmeans_get_assignments(self._h, ct.c_void_p(out.data_ptr()), on_dev))
            else:
                C.check(C.lib().kmeans_get_assignments(self._h, ct.c_void_p(out.ctypes.data), 0))
            return out
        a = np.empty(self.n, np.int32)
        C.check(C.lib().kmeans_get_assignments(self._h, ct.c_void_p(a.ctypes.data), 0))
        return a

    def bounds(self) -> np.ndarray:
        """fp32[n_local] MTI upper bounds u(x) after the last pass (caller order; verification)."""
        u = np.empty(self.n, np.float32)
        C.check(C.lib().kmeans_get_bounds(self._h, ct.c_void_p(u.ctypes.data), 0))
        return u

    def centroids(self) -> np.ndarray:
        c = np.empty((self.k, self.d), np.float64)
        C.check(C.lib().kmeans_get_centroids(self._h, ct.c_void_p(c.ctypes.data)))
        return c

    def set_centroids(self, cent) -> None:
        c = np.ascontiguousarray(cent, dtype=np.float64).reshape(self.k, self.d)
        C.check(C.lib().kmeans_set_centroids(self._h, ct.c_void_p(c.ctypes.data)))

    def sse(self) -> float:
        v = ct.c_double()
        C.check(C.lib().kmeans_sse(self._h, ct.byref(v)))
        return v.value

    def stats(self):
        cnt = ct.c_int32()
        C.check(C.lib().kmeans_get_stats(self._h, None, 0, ct.byref(cnt)))
        arr = (C.KmIterStats * max(1, cnt.value))()
        C.check(C.lib().kmeans_get_stats(self._h, arr, cnt.value, ct.byref(cnt)))
        return [{f: getattr(arr[i], f) for f, _ in C.KmIterStats._fields_} for i in range(cnt.value)]

    @property
    def launch_count(self) -> int:
        return int(C.lib().kmeans_launch_count(self._h))

    @property
    def device_bytes(self) -> int:
        """Device memory held by the context (bytes)."""
        return int(C.lib().kmeans_device_bytes(self._h))

    @property
    def engine(self) -> str:
        """Kernel of the MTI assignment pass ("k_walk", "k_mti_tc", "k_assign", "k_assign_dense")."""
        return C.lib().kmeans_engine(self._h).decode()

    def close(self) -> None:
        if getattr(self, "_h", None):
            C.lib().kmeans_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def seed_plusplus(points, k: int, uniforms, first_index: int, *, device: Optional[int] = None, stream=None):
    """k-means++ D² seeding (Eq. 2) through ``kmeans_seed_plusplus``: returns
    (chosen int64[k] row indices, centroids fp64 k x d).  ``uniforms``: k-1 draws in [0,1)."""
    L = C.lib()
    on_host = 1
    dev = 0 if device is None else device
    try:
        import torch
        if isinstance(points, torch.Tensor):
            if points.dtype != torch.float32 or not points.is_contiguous():
                raise ValueError("points must be a contiguous float32 tensor")
            if points.is_cuda:
                on_host = 0
                dev = points.device.index if device is None else device
                if stream is None:
                    stream = torch.cuda.current_stream(dev).cuda_stream
            else:
                points = points.numpy()
    except ImportError:
        pass
    if on_host:
        points = np.ascontiguousarray(points, dtype=np.float32)
        ptr = points.ctypes.data
    else:
        ptr = points.data_ptr()
    n, d = points.shape
    u = np.ascontiguousarray(uniforms, dtype=np.float64).reshape(-1)
    if u.size < k - 1:
        raise ValueError("need k-1 uniforms")
    chosen = np.empty(k, np.int64)
    cent = np.empty((k, d), np.float64)
    C.check(L.kmeans_seed_plusplus(int(n), int(d), int(k), ct.c_void_p(ptr), on_host, int(first_index),
                                   ct.c_void_p(u.ctypes.data), int(dev),
                                   ct.c_void_p(int(stream) if stream is not None else 0),
                                   ct.c_void_p(chosen.ctypes.data), ct.c_void_p(cent.ctypes.data)))
    return chosen, cent


def kmeanspp_multirun(points, k: int, runs, max_iters: int, tol: int = 0, *, prune: str = "mti",
                      device: Optional[int] = None):
    """k-means++ as PAPER.md §4.3 describes it (lines 1141-1149): r runs, each seeded by D²
    sampling (Eq. 2) and refined by Lloyd's (here the MTI engine), keeping the run with the
    smallest SSE (ties: the earlier run).  ``runs``: a list of (first_index, uniforms[k-1]).
    Returns (best run index, assignments, centroids, SSE, iterations)."""
    best = None
    for i, (first, u) in enumerate(runs):
        _, C0 = seed_plusplus(points, k, u, first, device=device)
        with KMeans(points, C0, prune=prune, device=device) as km:
            it, _ = km.run(max_iters, tol)
            sse = km.sse()
            if best is None or sse < best[3]:
                best = (i, km.assignments(), km.centroids(), sse, it)
    return best
