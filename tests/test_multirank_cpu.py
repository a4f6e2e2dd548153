"""N > 1 host logic on CPU with torch.distributed/gloo (world_size 2): the contiguous row
sharding (§7, 1538-1564), the unique-id broadcast, max-over-ranks timing, and the
sharded reduction math (per-rank partial sums + one allreduce == the unsharded oracle)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_1902_09527_b200.dist import broadcast_bytes, max_over_ranks, shard_bounds, sum_over_ranks
        from synth import make_config, make_points
        X, idx, _ = make_config("c2")
        n, k = X.shape[0], 100
        lo, hi = shard_bounds(n, rank, world)
        Xs = make_points("c2", rows=(lo, hi))              # a rank generates only its shard
        assert np.array_equal(Xs, X[lo:hi])
        payload = bytes(range(128)) if rank == 0 else b"\0" * 128
        got = broadcast_bytes(payload)
        assert got == bytes(range(128))
        assert max_over_ranks(float(rank + 1)) == float(world)
        assert sum_over_ranks(1.0) == float(world)
        # one Lloyd step, sharded: local assignment + local partial sums, then allreduce
        C0 = X[idx].astype(np.float64)
        a, _, _ = oracle.assign_brute(Xs, C0)
        sums, counts = oracle.cluster_sums(Xs, a, k)
        buf = torch.from_numpy(np.concatenate([sums.ravel(), counts.astype(np.float64)]))
        dist.all_reduce(buf)
        gs = buf[:k * 16].numpy().reshape(k, 16)
        gc = buf[k * 16:].numpy().astype(np.int64)
        C1, _ = oracle.update(gs, gc, C0)
        q.put((rank, C1, int(gc.sum())))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_shard_step():
    import oracle
    from synth import make_config
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    res = sorted([q.get() for _ in range(world)], key=lambda t: t[0])
    X, idx, _ = make_config("c2")
    C0 = X[idx].astype(np.float64)
    a, _, _ = oracle.assign_brute(X, C0)
    sums, counts = oracle.cluster_sums(X, a, 100)
    C1, _ = oracle.update(sums, counts, C0)
    for rank, C1r, total in res:
        assert total == X.shape[0]
        assert np.max(np.abs(C1r - C1)) <= 1e-13 * np.max(np.abs(C1))
    assert np.array_equal(res[0][1], res[1][1])       # identical on every rank


def test_shard_bounds_cover():
    from paper_1902_09527_b200.dist import shard_bounds
    for n in (1, 7, 65_608_366, 100_000_000):
        for G in (1, 2, 3, 4, 8):
            b = [shard_bounds(n, r, G) for r in range(G)]
            assert b[0][0] == 0 and b[-1][1] == n
            assert all(b[i][1] == b[i + 1][0] for i in range(G - 1))
            assert max(h - l for l, h in b) - min(h - l for l, h in b) <= 1


def test_bench_launcher_starts_n_ranks():
    """`bench.py --gpus 2` without a torchrun environment starts 2 ranks itself
    (torch.distributed.run on 127.0.0.1); on the reference arm rank 0 alone prints one JSON line
    with n_gpus = 2 and rank 1 exits 0 without work.  A WORLD_SIZE that contradicts --gpus fails."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--gpus", "2",
                          "--config", "c1", "--steps", "2", "--warmup", "1"],
                         capture_output=True, text=True, env=env, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    j = json.loads(lines[0])
    assert j["impl"] == "reference" and j["n_gpus"] == 2 and j["steps"] == 2
    bad = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--gpus", "2"],
                         capture_output=True, text=True, env=dict(env, WORLD_SIZE="1"), timeout=120)
    assert bad.returncode != 0
