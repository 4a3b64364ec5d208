"""Multi-GPU plumbing of the batched path: the instances of a
batch are independent, so rank r of W solves its own contiguous shard of
instances on its own GPU with no collective on the data path. torch.distributed
is used only for the timing reduction (max over ranks) and, where a caller
wants the whole batch on one rank, a gather of the solutions afterwards.

Two sharding modes:
  weak   every rank gets `per_rank` instances: instances
         [rank * per_rank, (rank + 1) * per_rank) of the seeded generator
         (bench.py: per-GPU work fixed as N grows)
  strong a fixed `total` split into balanced contiguous ranges
"""
from __future__ import annotations

import numpy as np

from . import synth
from .ocp import EqOCPBatch, EqSolutionBatch


def shard_bounds(total: int, rank: int, world: int) -> tuple[int, int]:
    """Balanced contiguous range (start, count) of `total` items for `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("rank out of range")
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


def generate_shard(cfg_idx: int, seed: int, rank: int, world: int, per_rank: int | None = None,
                   total: int | None = None, N: int | None = None) -> tuple[EqOCPBatch, int]:
    """This rank's instances of config `cfg_idx`; returns (batch, first index)."""
    if (per_rank is None) == (total is None):
        raise ValueError("give exactly one of per_rank (weak) or total (strong)")
    if per_rank is not None:
        start, count = rank * per_rank, per_rank
    else:
        start, count = shard_bounds(total, rank, world)
    return synth.generate(cfg_idx, seed=seed, batch=count, N=N, start=start), start


def max_over_ranks(x: float, device=None) -> float:
    """Max of a per-rank scalar (device timings: the job is as slow as its
    slowest rank)."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_solutions(sol: EqSolutionBatch, dst: int = 0) -> EqSolutionBatch | None:
    """Concatenate every rank's solution shard (in rank order) on `dst`."""
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size() == 1:
        return sol
    parts = [None] * dist.get_world_size() if dist.get_rank() == dst else None
    local = tuple(np.asarray(getattr(sol, k)) for k in ("u", "x", "lam"))
    dist.gather_object(local, parts, dst=dst)
    if dist.get_rank() != dst:
        return None
    return EqSolutionBatch(*[np.concatenate([p[i] for p in parts]) for i in range(3)])
