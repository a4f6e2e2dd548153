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
SRCS = [os.path.join(PKG, "csrc", f) for f in ("km_kernels.cu", "km_tc.cu", "km_walk.cu", "km_screen.cu", "km_tcc.cu", "km_ti.cu", "km_seed.cu", "km_api.cu")]
DEPS = SRCS + [os.path.join(PKG, "csrc", "km_device.cuh"), os.path.join(PKG, "csrc", "km_walk_body.cuh"), os.path.join(PKG, "csrc", "km_walk_common.cuh"), os.path.join(PKG, "csrc", "km_tc_common.cuh"), os.path.join(PKG, "csrc", "km_kernels.cuh"), os.path.join(ROOT, "include", "kmeans_b200.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def needs_build() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    return any(os.path.getmtime(f) > t for f in DEPS)


def _compile(src: str, obj: str, defines, verbose: bool):
    cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-c",
           "-I", os.path.join(ROOT, "include"), *[f"-D{x}" for x in defines], "-o", obj, src]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines=()) -> str:
    """Compile the library (``out``/``defines``: an A/B variant, see tools/build_variant.py).
    Each .cu is compiled to its own object in parallel (objects of unchanged sources are kept),
    then linked with cudart static."""
    from concurrent.futures import ThreadPoolExecutor
    so = out or SO
    if out is None and not force and not needs_build():
        return SO
    tag = "default" if out is None and not defines else "v" + str(abs(hash((so, tuple(defines)))) % 10**8)
    objdir = os.path.join(ROOT, "build", tag)
    os.makedirs(objdir, exist_ok=True)
    hdrs = [f for f in DEPS if not f.endswith(".cu")]
    newest_hdr = max(os.path.getmtime(f) for f in hdrs)
    jobs = []
    objs = []
    for src in SRCS:
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        objs.append(obj)
        if force or not os.path.exists(obj) or os.path.getmtime(obj) < max(os.path.getmtime(src), newest_hdr):
            jobs.append((src, obj))
    with ThreadPoolExecutor(max(1, min(len(jobs), os.cpu_count() or 1))) as ex:
        for f in [ex.submit(_compile, s_, o_, defines, verbose) for s_, o_ in jobs]:
            f.result()
    subprocess.check_call([NVCC, *ARCH, "-shared", "-o", so + ".tmp", *objs, "-ldl"])
    os.replace(so + ".tmp", so)
    return so


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(SO)
