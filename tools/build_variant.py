"""Build an A/B variant of the library with extra -D defines into variants/NAME.so.

    python tools/build_variant.py NAME [DEFINE ...]      e.g.  t640 KM_WALK_T8=640
Run it on the GPU box with  KM_LIB=variants/NAME.so python bench.py ...
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1902_09527_b200 import build as B  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
os.makedirs(os.path.join(ROOT, "variants"), exist_ok=True)
print(B.build(out=os.path.join(ROOT, "variants", name + ".so"), defines=defs))
