"""Build an A/B variant of the library with extra -D defines into variants/NAME.so.

    python tools/build_variant.py NAME [--only SRC.cu,...] [DEFINE ...]   e.g.  t640 KM_WALK_T8=640
--only: recompile just those sources with the defines and link them with the default build's
other objects (build/default, from the in-tree build).
Run it on the GPU box with  KM_LIB=variants/NAME.so python bench.py ...
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1902_09527_b200 import build as B  # noqa: E402

name, args = sys.argv[1], sys.argv[2:]
only = None
if args and args[0] == "--only":
    only, args = args[1].split(","), args[2:]
os.makedirs(os.path.join(ROOT, "variants"), exist_ok=True)
out = os.path.join(ROOT, "variants", name + ".so")
if only is None:
    print(B.build(out=out, defines=args))
else:
    objdir = os.path.join(ROOT, "build", "v_" + name)
    os.makedirs(objdir, exist_ok=True)
    objs = []
    for src in B.SRCS:
        base = os.path.basename(src)
        if base in only:
            obj = os.path.join(objdir, base + ".o")
            B._compile(src, obj, args, False)
        else:
            obj = os.path.join(ROOT, "build", "default", base + ".o")
        objs.append(obj)
    subprocess.check_call([B.NVCC, *B.ARCH, "-shared", "-o", out, *objs, "-ldl"])
    print(out)
