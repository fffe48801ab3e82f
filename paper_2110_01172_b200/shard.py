"""Batch sharding for independent transforms across GPUs.

Batched 2D transforms (BASELINE configs[4]: 512 x 2048^2 fp32) are independent
objects: each of N ranks (one process per GPU, torchrun) owns a contiguous
slice of the batch, runs its own plan on its own stream, and no data-path
collective exists. The only cross-rank traffic is the benchmark's barrier and
max-over-ranks timing reduction.
"""
from __future__ import annotations


def shard_range(total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced [start, stop) slice of `total` items for `rank`."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("need 0 <= rank < world")
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    stop = start + base + (1 if rank < extra else 0)
    return start, stop


def spot_check_indices(total: int, world: int) -> list[int]:
    """Items checked against the oracle: 0, every shard boundary, and the last."""
    idx = {0, total - 1}
    for r in range(world):
        s, e = shard_range(total, world, r)
        if e > s:
            idx.update((s, e - 1))
    return sorted(i for i in idx if 0 <= i < total)


def item_seed(global_index: int, base: int = 5) -> int:
    """Per-image seed (configs[4] uses seed 5 + image index)."""
    return base + global_index
