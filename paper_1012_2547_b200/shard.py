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


def gather_positions(local, group=None, device=None):
    """Every rank's int64 positions (rank order == position order) -> the global
    ascending position tensor on every rank: one all_gather of the counts, one
    all_gather of the count-padded slices (NCCL over NVLink on GPUs)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    local = torch.as_tensor(local, dtype=torch.int64)
    if device is not None:
        local = local.to(device)
    _, total, counts = exchange_counts(int(local.numel()), group, local.device)
    width = max(max(counts), 1)
    padded = torch.zeros(width, dtype=torch.int64, device=local.device)
    padded[: local.numel()] = local
    parts = [torch.empty_like(padded) for _ in range(world)]
    dist.all_gather(parts, padded, group=group)
    out = torch.cat([p[:c] for p, c in zip(parts, counts)])
    assert out.numel() == total
    return out


def pattern_range(K: int, world: int, rank: int) -> tuple[int, int]:
    """Batched mode: patterns [k0, k1) of this rank; the text
    is replicated, so no halo and no position exchange inside the search."""
    return K * rank // world, K * (rank + 1) // world


def sharded_search_batch(patterns, text, batch_searcher, group=None, device=None):
    """Batched mode over ranks: rank r runs `batch_searcher(patterns[k0:k1], text)
    -> (positions, offsets[k1-k0+1])` on the full text for its pattern range; the
    CSR pieces are gathered into the whole batch's CSR (positions, offsets[K+1])
    on every rank, in pattern order."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    K = len(patterns)
    k0, k1 = pattern_range(K, world, rank)
    if k1 > k0:
        pos, offs = batch_searcher(patterns[k0:k1], text)
        pos = torch.as_tensor(pos, dtype=torch.int64)
        per = torch.as_tensor(offs, dtype=torch.int64).diff()
    else:
        pos = torch.zeros(0, dtype=torch.int64)
        per = torch.zeros(0, dtype=torch.int64)
    if device is not None:
        pos, per = pos.to(device), per.to(device)
    # per-pattern counts of every rank, padded to the widest range
    width = max(K // world + 1, 1)
    pc = torch.zeros(width, dtype=torch.int64, device=pos.device)
    pc[: per.numel()] = per
    parts = [torch.empty_like(pc) for _ in range(world)]
    dist.all_gather(parts, pc, group=group)
    counts = torch.cat([parts[r][: pattern_range(K, world, r)[1] - pattern_range(K, world, r)[0]]
                        for r in range(world)])
    offsets = torch.zeros(K + 1, dtype=torch.int64, device=pos.device)
    offsets[1:] = torch.cumsum(counts, 0)
    allpos = gather_positions(pos, group, pos.device)
    return allpos, offsets
