import time, sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from synth import make_config
from paper_1902_09527_b200 import KMeans
X, idx, _ = make_config("c3")
C0 = X[idx].astype(np.float64)
Xh = torch.empty(X.shape, dtype=torch.float32, pin_memory=True); Xh.numpy()[:] = X
torch.cuda.synchronize()
for rep in range(2):
    t0 = time.perf_counter()
    km = KMeans(Xh, C0, prune="mti", device=0)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    km.iterate(); t2 = time.perf_counter()
    for _ in range(29): km.iterate()
    t3 = time.perf_counter()
    a = km.assignments(); t4 = time.perf_counter()
    C = km.centroids(); t5 = time.perf_counter()
    km.close(); t6 = time.perf_counter()
    print(f"rep{rep}: create {1e3*(t1-t0):.1f} ms, iter1 {1e3*(t2-t1):.1f}, 29 iters {1e3*(t3-t2):.1f}, assignments {1e3*(t4-t3):.1f}, centroids {1e3*(t5-t4):.1f}, close {1e3*(t6-t5):.1f}")
