"""Batch-sharded multi-GPU inference.

Samples are independent, so the reference's virtual-block partition
(engine.py:53-61: output channel x sample group) coarsens to "each rank owns a
contiguous slice of the batch".  Weights (CSR packs) are replicated per rank;
nothing is exchanged on the hot path; the only collective is the optional
final gather of the per-rank outputs (one all_gather of the logits/features).
"""

from __future__ import annotations


def shard_range(n: int, rank: int, world: int, align: int = 1) -> tuple[int, int]:
    """[start, stop) of rank's samples: contiguous, balanced, start/stop multiples of
    `align` (32 keeps BI32 sample blocks whole) except for the last rank."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    if n < 0:
        raise ValueError("negative batch")
    units = (n + align - 1) // align
    base, extra = divmod(units, world)
    u0 = rank * base + min(rank, extra)
    u1 = u0 + base + (1 if rank < extra else 0)
    return min(n, u0 * align), min(n, u1 * align)


def shard_sizes(n: int, world: int, align: int = 1) -> list[int]:
    return [b - a for a, b in (shard_range(n, r, world, align) for r in range(world))]


def gather_shards(local, n: int, group=None, align: int = 1):
    """Concatenate every rank's rows (dim 0) in rank order on every rank.

    Uses torch.distributed (NCCL on GPUs, gloo on CPU).  Shards may be uneven:
    they are padded to the largest shard for the all_gather and trimmed."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    sizes = shard_sizes(n, world, align)
    mx = max(sizes)
    if local.shape[0] != sizes[dist.get_rank(group)]:
        raise ValueError(f"local shard has {local.shape[0]} rows, expected "
                         f"{sizes[dist.get_rank(group)]}")
    pad = torch.zeros((mx,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[:local.shape[0]] = local
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    return torch.cat([b[:s] for b, s in zip(bufs, sizes)], dim=0)
