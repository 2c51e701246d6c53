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


class ShardedRun:
    """One rank's view of a batch-sharded inference job.

    ``global_batch`` samples are split into contiguous per-rank slices
    (``shard_range``); each rank runs ``forward`` (its own replica of the
    network: CSR packs replicated, no exchange on the hot path) over its slice
    and the per-rank outputs are concatenated in rank order by one final
    ``gather_shards``.  ``weak`` mode fixes the per-rank batch instead
    (``global_batch = world * per_rank``).  Mirrors the reference's partition of
    the work into independent virtual blocks (engine.py:53-61): sample groups
    never interact, so the gathered result equals the single-process one bit for
    bit."""

    def __init__(self, global_batch: int, rank: int = 0, world: int = 1, align: int = 1,
                 group=None):
        self.global_batch, self.rank, self.world, self.align = global_batch, rank, world, align
        self.group = group
        self.start, self.stop = shard_range(global_batch, rank, world, align)

    @classmethod
    def from_env(cls, global_batch: int, align: int = 1, group=None) -> "ShardedRun":
        """Rank and world size from torch.distributed when it is initialised (else 1 rank)."""
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            return cls(global_batch, dist.get_rank(group), dist.get_world_size(group), align, group)
        return cls(global_batch, 0, 1, align, group)

    @classmethod
    def weak(cls, per_rank: int, rank: int = 0, world: int = 1, group=None) -> "ShardedRun":
        return cls(per_rank * world, rank, world, per_rank, group)

    @property
    def local_batch(self) -> int:
        return self.stop - self.start

    def local(self, x):
        """This rank's rows of a global batch (dim 0)."""
        if x.shape[0] != self.global_batch:
            raise ValueError(f"global input has {x.shape[0]} rows, expected {self.global_batch}")
        return x[self.start:self.stop]

    def gather(self, local_out):
        """The final (and only) collective: every rank's output rows, in rank order."""
        if self.world == 1:
            if local_out.shape[0] != self.global_batch:
                raise ValueError("local output does not cover the batch")
            return local_out
        return gather_shards(local_out, self.global_batch, self.group, self.align)

    def run(self, x_global, forward):
        """gather(forward(local(x_global)))."""
        return self.gather(forward(self.local(x_global)))
