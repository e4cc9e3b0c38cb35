"""Multi-GPU sharding of one text: one process per GPU.

Rank r owns start positions [lo_r, hi_r) and reads text[lo_r : min(hi_r + m - 1, n)),
so the (m-1)-byte overlap never double-reports.  The only exchange is an
all_gather of per-rank counts, which turns rank-local results into slices of
one globally ordered output (rank order == position order).  Works with any
torch.distributed backend (NCCL on GPUs; gloo in the CPU tests).
"""
from __future__ import annotations


def shard_bounds(n: int, m: int, world: int, rank: int) -> tuple[int, int, int]:
    """(lo, hi, read_hi): starts [lo, hi) and bytes [lo, read_hi) for this rank."""
    if m > n:
        return 0, 0, 0
    starts = n - m + 1
    lo = starts * rank // world
    hi = starts * (rank + 1) // world
    return lo, hi, min(hi + m - 1, n) if hi > lo else lo


def exchange_counts(local_count: int, group=None, device=None) -> tuple[int, int, list[int]]:
    """all_gather of per-rank counts -> (global offset of this rank, total, counts)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    t = torch.tensor([local_count], dtype=torch.int64, device=device)
    allc = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(allc, t, group=group)
    counts = [int(x.item()) for x in allc]
    return sum(counts[:rank]), sum(counts), counts


def sharded_search(pattern: bytes, local_text, n: int, searcher, group=None, device=None):
    """Search this rank's shard with `searcher(pattern, bytes_or_tensor) -> int64
    array/tensor`; return (global positions of this rank, global offset, total)."""
    import torch.distributed as dist

    m = len(pattern)
    lo, hi, read_hi = shard_bounds(n, m, dist.get_world_size(group), dist.get_rank(group))
    if hi > lo:
        local = searcher(pattern, local_text) + lo
    else:
        local = searcher(pattern, local_text[:0])
    off, total, _ = exchange_counts(len(local), group, device)
    return local, off, total
