"""Multi-GPU plumbing for the filter-sharded workloads (one process per GPU).

C5-style batches shard by filter index with NO data-path collective
(SURVEY §8(e)): every rank runs its own filters; torch.distributed is used only
for the barrier around the timed region and the max-over-ranks time.
"""
from __future__ import annotations

import os


def env():
    """(rank, world, local_rank) from torchrun's environment."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def rank_seed(seed: int, rank: int) -> int:
    """Weak scaling: rank r runs its own batch of filters with a distinct seed."""
    return seed + 7919 * rank


def shard(batch: int, rank: int, world: int) -> tuple:
    """Strong scaling: contiguous filter range [lo, hi) of rank r (remainder spread over the first ranks)."""
    q, r = divmod(batch, world)
    lo = rank * q + min(rank, r)
    return lo, lo + q + (1 if rank < r else 0)


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar over the default process group (identity when not initialised)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
