"""CPU checks of the boundary: the library builds for sm_100a, loads, and exports every entry
point include/kmeans_b200.h declares (no compute calls without a GPU)."""
import ctypes as ct
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "kmeans_b200.h")


def declared():
    src = open(HDR).read()
    return sorted(set(re.findall(r"\b(kmeans_[a-z_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared()
    for must in ("kmeans_create", "kmeans_iterate", "kmeans_run", "kmeans_get_assignments",
                 "kmeans_get_centroids", "kmeans_set_centroids", "kmeans_sse", "kmeans_destroy",
                 "kmeans_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_1902_09527_b200 import _capi
    L = _capi.lib()
    for name in declared():
        assert hasattr(L, name), name
        assert name in _capi.SIGNATURES, name
    assert L.kmeans_version().startswith(b"kmeans_b200")
    assert L.kmeans_last_error() == b""


def test_library_is_sm100a():
    from paper_1902_09527_b200 import _capi
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _capi.SO_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_struct_layouts():
    from paper_1902_09527_b200 import _capi
    assert ct.sizeof(_capi.KmOptions) == 216
    assert ct.sizeof(_capi.KmIterStats) == 72
    o = _capi.KmOptions()
    _capi.lib().kmeans_default_options(ct.byref(o))
    assert o.world == 1 and o.prune == 0 and o.resort_fraction == 0.0 and o.engine == 0


def test_create_argument_errors_without_gpu():
    """Argument validation happens before any CUDA call."""
    import numpy as np
    from paper_1902_09527_b200 import KMeans, KMeansError
    with pytest.raises(KMeansError, match="KM_EARG"):
        KMeans(np.zeros((4, 2), np.float32), np.zeros((5, 2)))
    with pytest.raises(KMeansError, match="KM_EARG"):
        KMeans(np.zeros((4, 65), np.float32), np.zeros((2, 65)))
