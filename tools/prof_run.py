"""Small profiling driver: N iterations of the library on a config-shaped synthetic set.

    python tools/prof_run.py --config c3 --n 8000000 --iters 10 [--engine auto|cuda|tensor]
Prints per-iteration stats (kernel ms, dists, fallbacks) — for ncu / quick A-B timing.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1902_09527_b200 import KMeans  # noqa: E402
from synth import make_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--n", type=int, default=8_000_000)
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--engine", default="auto")
ap.add_argument("--resort", default="auto")
ap.add_argument("--resort-fraction", type=float, default=0.0)
args = ap.parse_args()
X, idx, _ = make_config(args.config, n=args.n)
C0 = X[idx].astype(np.float64)
Xd = torch.from_numpy(X).cuda()
with KMeans(Xd, C0, prune="mti", engine=args.engine, resort=args.resort,
            resort_fraction=args.resort_fraction) as km:
    for _ in range(args.iters):
        km.iterate()
    torch.cuda.synchronize()
    st = km.stats()
    print(f"sum ms_iter t=4..{len(st)}: {sum(s['ms_iter'] for s in st[3:]):.3f}")
    for i, s in enumerate(st):
        print(f"t={i + 1} ms_assign={s['ms_assign']:.3f} ms_iter={s['ms_iter']:.3f} ms_sort={s['ms_sort']:.3f} "
              f"changed={s['changed']} dists={s['dists']} clause1={s['clause1']} refined={s['refined']} "
              f"steps={s['walk_steps']} resorted={s['resorted']}")
