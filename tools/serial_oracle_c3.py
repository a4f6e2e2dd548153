"""One serial (1 thread) knori- iteration of the fp64 oracle on the full C3 data set, at k = 10 and
k = 100, to set beside the paper's serial table (Table "baseline": knori- 7.49 s
per iteration on Friendster-8, every distance computed).  Test/measurement infrastructure: calls
only oracle/ and synth/.  usage: python tools/serial_oracle_c3.py [out.json]"""
import json
import os
import platform
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
from synth import make_config  # noqa: E402


def main():
    X, idx, _ = make_config("c3")
    oracle.set_threads(1)
    out = {"config": "c3", "n": int(X.shape[0]), "d": int(X.shape[1]), "threads": oracle.num_threads(),
           "cpu": platform.processor() or platform.machine(), "paper_knori_minus_s_per_iter": 7.49,
           "paper_ref": "PAPER.md:566-595 (Friendster-8, 1 thread, all distances)", "iterations": []}
    for k in (10, 100):
        C0 = X[idx[:k]].astype(np.float64)
        t0 = time.perf_counter()
        a, _, _ = oracle.assign_brute(X, C0)          # every distance (knori-)
        t1 = time.perf_counter()
        sums, counts = oracle.cluster_sums(X, a, k)
        C1, _ = oracle.update(sums, counts, C0)
        t2 = time.perf_counter()
        out["iterations"].append({"k": k, "s_per_iter": t2 - t0, "assign_s": t1 - t0, "sums_update_s": t2 - t1})
        print(json.dumps(out["iterations"][-1]), flush=True)
    if len(sys.argv) > 1:
        json.dump(out, open(sys.argv[1], "w"), indent=1)


if __name__ == "__main__":
    main()
