"""Time k-means++ D² seeding (kmeans_seed_plusplus) at a config's full size on one GPU, next to the
oracle on a row sample.  usage: python tools/pp_bench.py [--config c3] [--reps 3]"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1902_09527_b200 import seed_plusplus  # noqa: E402
from synth import make_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()
X, _, spec = make_config(args.config)
k = spec["k"]
u = np.random.default_rng(17).random(k - 1)
Xd = torch.from_numpy(X).cuda()
seed_plusplus(Xd, k, u, 0)
torch.cuda.synchronize()
ts = []
for _ in range(args.reps):
    t0 = time.perf_counter()
    seed_plusplus(Xd, k, u, 0)
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
import oracle  # noqa: E402
m = min(X.shape[0], 1_000_000)
t0 = time.perf_counter()
oracle.seed_plusplus(X[:m], k, u, 0)
to = (time.perf_counter() - t0) * X.shape[0] / m
out = {"what": "k-means++ D^2 seeding (kmeans_seed_plusplus)", "config": f"{args.config}: n={X.shape[0]}, d={X.shape[1]}, k={k}",
       "gpu_s": min(ts), "gpu_s_all": ts, "oracle_s_extrapolated": to,
       "oracle_sample": f"first {m} rows, extrapolated by rows (1 host thread, numpy)",
       "bytes_per_round": int(X.shape[0]) * (4 * X.shape[1] + 16)}
print(json.dumps(out))
