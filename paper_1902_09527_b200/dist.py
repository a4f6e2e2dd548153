"""Multi-GPU plumbing (one process per GPU, torch.distributed for bootstrap only).

Sharding (§7, 1538-1564: each machine processes its local data and global state is
merged; no inter-machine load balancing, 1547-1553): rank r of G owns the contiguous rows
[floor(r n / G), floor((r+1) n / G)).  The library's own NCCL communicator performs the one
allreduce per iteration; torch.distributed only ships the ncclUniqueId and takes the
max-over-ranks of timings.
"""
from __future__ import annotations

import os


def shard_bounds(n: int, rank: int, world: int):
    return (n * rank) // world, (n * (rank + 1)) // world


def env_rank_world():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), \
        int(os.environ.get("LOCAL_RANK", "0"))


def broadcast_bytes(payload: bytes, src: int = 0) -> bytes:
    """Broadcast a small byte string from ``src`` with the default process group."""
    import torch
    import torch.distributed as dist
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else torch.device("cpu")
    t = torch.zeros(len(payload) if payload else 128, dtype=torch.uint8, device=dev)
    if dist.get_rank() == src:
        t.copy_(torch.frombuffer(bytearray(payload), dtype=torch.uint8))
    dist.broadcast(t, src)
    return bytes(t.cpu().numpy().tobytes())


def max_over_ranks(value: float) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return value
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else torch.device("cpu")
    t = torch.tensor([value], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return value
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else torch.device("cpu")
    t = torch.tensor([value], dtype=torch.float64, device=dev)
    dist.all_reduce(t)
    return float(t.item())
