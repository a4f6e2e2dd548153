"""Write the full-size oracle trajectories of C3, C4 and C5 to tests/golden/ (traj_<cfg>.json
plus traj_<cfg>_C.npy and traj_<cfg>_asample.npy).

Calls only ``oracle/`` (fp64, MTI mode, validated lossless against brute force by
tests/test_oracle_pins.py) and ``synth/`` (the seeded inputs); nothing here comes from the CUDA
path.  Per iteration t it records changed, dists (MTI semantics), clause1, empty clusters,
SSE_t = sum ||x - C_t[a_t]||^2 and sha256(a_t as int32 bytes, caller row order); it stores
every C_t (fp64, T x k x d) and a_T at rows 0, 1024, 2048, ... (diagnostics for mismatch counts).

    OMP_NUM_THREADS=8 python tools/make_golden.py c3 c4 c5
"""
from __future__ import annotations

import hashlib
import json
import os
import platform
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from synth import CONFIGS, make_config, sha256_points  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")
SAMPLE_STRIDE = 1024


def a_sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, np.int32).tobytes()).hexdigest()


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def run(name: str) -> None:
    spec = CONFIGS[name]
    t0 = time.time()
    X, idx, man = make_config(name)
    gen_s = time.time() - t0
    C0 = X[idx].astype(np.float64)
    Cs, per = [], []
    tick = [time.time()]

    def on_iter(t, a, C, rec):
        now = time.time()
        rec = dict(rec, a_sha256=a_sha(a), seconds=round(now - tick[0], 3))
        per.append(rec)
        Cs.append(C.copy())
        tick[0] = time.time()
        print(f"[{name}] t={t} changed={rec['changed']} dists={rec['dists']} clause1={rec['clause1']} "
              f"empty={rec['empty']} sse={rec['sse']:.12e} {rec['seconds']} s", flush=True)

    r = oracle.lloyd_trace(X, C0, spec.max_iters, spec.tol, "mti", on_iter=on_iter)
    out = dict(config=name, n=int(X.shape[0]), d=spec.d, k=spec.k, max_iters=spec.max_iters, tol=spec.tol,
               sha256_X=sha256_points(X), forgy_head=idx[:8].tolist(), mode="mti",
               iterations=r.iterations, final_sse=r.final_sse, final_a_sha256=per[-1]["a_sha256"],
               sample_stride=SAMPLE_STRIDE, per_iter=per,
               producer=dict(script="tools/make_golden.py", oracle="oracle.lloyd_trace (mode=mti)",
                             threads=oracle.num_threads(), cpu=cpu_model(), numpy=np.__version__,
                             generation_s=round(gen_s, 1)))
    with open(os.path.join(GOLD, f"traj_{name}.json"), "w") as f:
        json.dump(out, f, indent=1)
    np.save(os.path.join(GOLD, f"traj_{name}_C.npy"), np.stack(Cs))
    np.save(os.path.join(GOLD, f"traj_{name}_asample.npy"), r.a[::SAMPLE_STRIDE].astype(np.int16))
    print(f"[{name}] done: {r.iterations} iterations, {time.time() - t0:.0f} s", flush=True)


if __name__ == "__main__":
    for nm in sys.argv[1:] or ["c3", "c4", "c5"]:
        run(nm)
