"""oracle.lloyd_trace (the per-iteration driver the full-size golden trajectories come from)
is the C loop oracle_lloyd step for step: bitwise-equal outputs on C1 and C2 in both modes."""
import numpy as np
import pytest

import oracle
from synth import make_config


@pytest.mark.parametrize("name,iters", [("c1", 100), ("c2", 12)])
@pytest.mark.parametrize("mode", ["brute", "mti"])
def test_trace_equals_lloyd(name, iters, mode):
    X, idx, _ = make_config(name)
    C0 = X[idx].astype(float)
    seen = []
    r = oracle.lloyd(X, C0, iters, 0, mode)
    q = oracle.lloyd_trace(X, C0, iters, 0, mode, on_iter=lambda t, a, C, rec: seen.append(t))
    assert q.iterations == r.iterations and seen == list(range(1, r.iterations + 1))
    assert np.array_equal(q.a, r.a) and np.array_equal(q.C, r.C)
    for f in ("changed", "dists", "clause1", "empty", "sse"):
        assert np.array_equal(getattr(q, f), getattr(r, f)), f
