"""Pair-level data parallelism across GPUs.

Registrations of distinct pairs are independent (reference SPEC.md:400), so
the multi-GPU path shards whole pairs across ranks with no data-path
collective: rank r of N owns the queue of seeds r, r+N, ... of the job.  torch.distributed is only
used to align timing windows (barrier) and to take the max of the per-rank
device times, as the benchmark contract requires.
"""

from __future__ import annotations

import os

__all__ = ["RankInfo", "rank_info", "shard_seeds", "weak_seeds", "job_throughput",
           "max_over_ranks", "sum_over_ranks", "barrier"]


class RankInfo:
    def __init__(self, rank, world, local):
        self.rank, self.world, self.local = rank, world, local

    def __repr__(self):
        return f"RankInfo(rank={self.rank}, world={self.world}, local={self.local})"


def rank_info(env=None):
    """RANK / WORLD_SIZE / LOCAL_RANK as set by torch.distributed.run."""
    env = os.environ if env is None else env
    return RankInfo(int(env.get("RANK", "0")), int(env.get("WORLD_SIZE", "1")),
                    int(env.get("LOCAL_RANK", "0")))


def shard_seeds(rank, world, total):
    """Strong scaling (BASELINE config 4 as written): the job is `total`
    pairs, seeds 0..total-1, and rank r of `world` owns seeds r, r+world,
    r+2*world, ... — disjoint queues that together cover the job once."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside a world of {world}")
    return list(range(rank, total, world))


def weak_seeds(rank, per_rank):
    """Weak scaling (reported as an extra only): rank r registers its own
    `per_rank` pairs, seeds r*per_rank .. r*per_rank + per_rank - 1."""
    return [rank * per_rank + i for i in range(per_rank)]


def job_throughput(px_iters, seconds, world=1, device=None):
    """Whole-job Mpx*iter/s: the px*iter of ALL ranks (summed over the
    process group) over the job's time (the max over ranks, taken by the
    caller)."""
    return sum_over_ranks(float(px_iters), world, device) / seconds / 1e6


def sum_over_ranks(value, world, device=None):
    """Sum of a per-rank scalar over the default process group."""
    if world <= 1:
        return float(value)
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64,
                     device=device if device is not None else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def max_over_ranks(value, world, device=None):
    """Max of a per-rank scalar over the default process group."""
    if world <= 1:
        return float(value)
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64,
                     device=device if device is not None else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
