"""Pair-level data parallelism across GPUs.

Registrations of distinct pairs are independent (reference SPEC.md:400), so
the multi-GPU path shards whole pairs across ranks with no data-path
collective: rank r of N owns its own pair queue.  torch.distributed is only
used to align timing windows (barrier) and to take the max of the per-rank
device times, as the benchmark contract requires.
"""

from __future__ import annotations

import os

__all__ = ["RankInfo", "rank_info", "shard_seeds", "job_throughput", "max_over_ranks",
           "barrier"]


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


def shard_seeds(rank, pairs_per_rank, available=None):
    """Seeds of rank's pair queue (weak scaling: every rank registers its own
    `pairs_per_rank` pairs, seeds rank*P .. rank*P+P-1).  When `available`
    (the seeds with cached meshes) is given, seeds outside it are replaced by
    seed % len(available) — replicas of cached pairs; the caller reports it."""
    seeds = [rank * pairs_per_rank + i for i in range(pairs_per_rank)]
    if available is None:
        return seeds, seeds
    avail = sorted(available)
    used = [s if s in available else avail[s % len(avail)] for s in seeds]
    return seeds, used


def job_throughput(px_iters_per_rank, seconds, world):
    """Whole-job Mpx*iter/s: every rank processed the same amount of work in
    at most `seconds` (the max over ranks)."""
    return world * float(px_iters_per_rank) / seconds / 1e6


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
