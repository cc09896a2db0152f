"""Multi-GPU shard launcher logic (layer L4): one process per GPU, contiguous
shards, no collective on the data path.  Elements are independent (the
primality of N[i] depends on N[i] only), so the array
partitions with no exchange step; torch.distributed (NCCL on GPUs, gloo in the
CPU tests) only reduces the per-rank prime count for validation and the
per-rank time for reporting."""
from __future__ import annotations


def strong_shard(rank: int, world: int, n: int) -> tuple[int, int]:
    """[lo, hi) of a fixed array of n elements owned by `rank` of `world`:
    lo = floor(r n / W), hi = floor((r + 1) n / W).  Shards cover [0, n)
    exactly once and differ in size by at most one element."""
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    return (rank * n) // world, ((rank + 1) * n) // world


def weak_shard(rank: int, world: int, n_per_rank: int) -> tuple[int, int]:
    """[lo, hi) of the generator index space owned by `rank` when every rank
    classifies a full batch of n_per_rank elements (weak scaling)."""
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    return rank * n_per_rank, (rank + 1) * n_per_rank


def value_range_shard(rank: int, world: int, lo: int, hi: int) -> tuple[int, int]:
    """[a, b) of the VALUE range [lo, hi) owned by `rank` when a dense range
    N = lo, lo+1, ..., hi-1 is split across ranks (config C4):
    a = lo + floor(r (hi - lo) / W).  Each rank builds its input as a device
    iota and its plan sieves only its own window [a, b) (2^32 / W values)."""
    a, b = strong_shard(rank, world, hi - lo)
    return lo + a, lo + b


def reduce_count(count: int, device=None, group=None) -> int:
    """Sum of per-rank prime counts over the process group (validation)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([int(count)], dtype=torch.int64, device=device)
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return int(t.item())


def reduce_max(value: float, device=None, group=None) -> float:
    """Max over ranks (a multi-GPU time is the slowest rank's)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
