"""Build the sm_100a shared library ``libkmeans_b200.so`` in-tree with nvcc.

The library is the whole product path: CUDA kernels (``csrc/km_kernels.cu``) and the C-ABI
runtime (``csrc/km_api.cu``, declared in ``include/kmeans_b200.h``).  cudart is linked
statically; NCCL is loaded with dlopen only when world > 1.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
SO = os.path.join(PKG, "libkmeans_b200.so")
SRCS = [os.path.join(PKG, "csrc", f) for f in ("km_kernels.cu", "km_tc.cu", "km_walk.cu", "km_seed.cu", "km_api.cu")]
DEPS = SRCS + [os.path.join(PKG, "csrc", "km_device.cuh"), os.path.join(PKG, "csrc", "km_kernels.cuh"), os.path.join(ROOT, "include", "kmeans_b200.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def needs_build() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    return any(os.path.getmtime(f) > t for f in DEPS)


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines=()) -> str:
    """Compile the library (``out``/``defines``: an A/B variant, see tools/build_variant.py)."""
    so = out or SO
    if out is None and not force and not needs_build():
        return SO
    cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
           "-I", os.path.join(ROOT, "include"), *[f"-D{x}" for x in defines], "-o", so + ".tmp", *SRCS, "-ldl"]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    os.replace(so + ".tmp", so)
    return so


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(SO)
