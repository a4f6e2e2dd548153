"""ctypes binding of ``libkmeans_b200.so`` (C ABI in ``include/kmeans_b200.h``).

Argument marshalling only: every step of the k-means iteration runs in the library's CUDA
kernels.  There is no CPU or PyTorch fallback — if the library is missing or cannot load,
``lib()`` raises.
"""
from __future__ import annotations

import ctypes as ct
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
# KM_LIB: an alternative build of the same library (A/B kernel variants, tools/build_variant.py)
SO_PATH = os.environ.get("KM_LIB") or os.path.join(_PKG, "libkmeans_b200.so")

KM_OK, KM_EARG, KM_ENONFINITE, KM_ECUDA, KM_ENCCL, KM_ENOMEM, KM_ESTATE = range(7)
KM_PRUNE_MTI, KM_PRUNE_NONE, KM_PRUNE_TI = 0, 1, 2
KM_RESORT_AUTO, KM_RESORT_NEVER, KM_RESORT_ALWAYS = 0, 1, 2
KM_ENGINE_AUTO, KM_ENGINE_CUDA_CORE, KM_ENGINE_TENSOR, KM_ENGINE_SCREEN, KM_ENGINE_TENSOR_SCREEN, KM_ENGINE_TENSOR_CHUNKED = 0, 1, 2, 3, 4, 5
STATUS_NAMES = {0: "KM_OK", 1: "KM_EARG", 2: "KM_ENONFINITE", 3: "KM_ECUDA", 4: "KM_ENCCL",
                5: "KM_ENOMEM", 6: "KM_ESTATE"}


class KmOptions(ct.Structure):
    _fields_ = [("device", ct.c_int32), ("stream", ct.c_void_p), ("prune", ct.c_int32),
                ("rank", ct.c_int32), ("world", ct.c_int32),
                ("nccl_unique_id", ct.c_uint8 * 128), ("n_global", ct.c_int64),
                ("check_finite", ct.c_int32), ("points_on_host", ct.c_int32),
                ("resort_policy", ct.c_int32), ("resort_fraction", ct.c_float),
                ("engine", ct.c_int32), ("spherical", ct.c_int32), ("no_graph", ct.c_int32),
                ("force_comm", ct.c_int32), ("resum_moves", ct.c_float), ("reserved", ct.c_int32 * 3)]


class KmIterStats(ct.Structure):
    _fields_ = [("changed", ct.c_int64), ("dists", ct.c_int64), ("clause1", ct.c_int64),
                ("refined", ct.c_int64), ("walk_steps", ct.c_int64), ("empty", ct.c_int32), ("resorted", ct.c_int32),
                ("ms_iter", ct.c_float), ("ms_assign", ct.c_float), ("ms_sort", ct.c_float),
                ("ms_comm", ct.c_float), ("fallbacks", ct.c_int64)]


# name -> (restype, argtypes); the list is also the export check of tests/test_capi_symbols.py
SIGNATURES = {
    "kmeans_default_options": (None, [ct.POINTER(KmOptions)]),
    "kmeans_nccl_unique_id": (ct.c_int32, [ct.POINTER(ct.c_uint8)]),
    "kmeans_create": (ct.c_int32, [ct.c_int64, ct.c_int32, ct.c_int32, ct.c_void_p, ct.c_void_p,
                                   ct.POINTER(KmOptions), ct.POINTER(ct.c_void_p)]),
    "kmeans_iterate": (ct.c_int32, [ct.c_void_p, ct.POINTER(ct.c_int64), ct.POINTER(ct.c_int64)]),
    "kmeans_finalize": (ct.c_int32, [ct.c_void_p]),
    "kmeans_run": (ct.c_int32, [ct.c_void_p, ct.c_int32, ct.c_int64, ct.POINTER(ct.c_int32),
                                ct.POINTER(ct.c_int64)]),
    "kmeans_get_assignments": (ct.c_int32, [ct.c_void_p, ct.c_void_p, ct.c_int32]),
    "kmeans_get_bounds": (ct.c_int32, [ct.c_void_p, ct.c_void_p, ct.c_int32]),
    "kmeans_get_centroids": (ct.c_int32, [ct.c_void_p, ct.c_void_p]),
    "kmeans_set_centroids": (ct.c_int32, [ct.c_void_p, ct.c_void_p]),
    "kmeans_sse": (ct.c_int32, [ct.c_void_p, ct.POINTER(ct.c_double)]),
    "kmeans_get_stats": (ct.c_int32, [ct.c_void_p, ct.POINTER(KmIterStats), ct.c_int32,
                                      ct.POINTER(ct.c_int32)]),
    "kmeans_seed_plusplus": (ct.c_int32, [ct.c_int64, ct.c_int32, ct.c_int32, ct.c_void_p, ct.c_int32,
                                          ct.c_int64, ct.c_void_p, ct.c_int32, ct.c_void_p, ct.c_void_p,
                                          ct.c_void_p]),
    "kmeans_launch_count": (ct.c_int64, [ct.c_void_p]),
    "kmeans_device_bytes": (ct.c_int64, [ct.c_void_p]),
    "kmeans_engine": (ct.c_char_p, [ct.c_void_p]),
    "kmeans_destroy": (None, [ct.c_void_p]),
    "kmeans_last_error": (ct.c_char_p, []),
    "kmeans_version": (ct.c_char_p, []),
}

_lib = None


class KMeansError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


def lib():
    """Load the in-tree library (raises if it was not built: run __graft_entry__.build())."""
    global _lib
    if _lib is None:
        if not os.path.exists(SO_PATH):
            raise ImportError(f"{SO_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ct.CDLL(SO_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(status: int) -> None:
    if status != KM_OK:
        raise KMeansError(status, lib().kmeans_last_error().decode(errors="replace"))
