"""World-size-2 gloo tests of the multi-GPU host logic (pair sharding, no
data-path collective, max-over-ranks timing), run on CPU."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1411_2141_b200 import pairqueue


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    info = pairqueue.rank_info()
    assert (info.rank, info.world) == (rank, world)
    seeds, used = pairqueue.shard_seeds(info.rank, 4, available=set(range(6)))
    # per-rank "device time": rank 1 is the slow one
    t = 1.0 + rank
    pairqueue.barrier(world)
    tmax = pairqueue.max_over_ranks(t, world)
    # everyone can gather the shards to check disjointness
    gathered = [None] * world
    dist.all_gather_object(gathered, seeds)
    out[rank] = (seeds, used, tmax, gathered,
                 pairqueue.job_throughput(10e6, tmax, world))
    dist.destroy_process_group()


def test_two_rank_pair_queue_gloo():
    world = 2
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    s0, u0, t0, g0, v0 = res[0]
    s1, u1, t1, g1, v1 = res[1]
    assert s0 == [0, 1, 2, 3] and s1 == [4, 5, 6, 7]
    assert not set(s0) & set(s1)                      # disjoint pair queues
    assert u1 == [4, 5, 0, 1]                         # replicas of cached seeds
    assert t0 == t1 == 2.0                            # max over ranks
    assert g0 == g1 == [s0, s1]
    assert v0 == v1 == pytest.approx(2 * 10e6 / 2.0 / 1e6)


def test_single_rank_defaults():
    info = pairqueue.rank_info({})
    assert (info.rank, info.world, info.local) == (0, 1, 0)
    assert pairqueue.max_over_ranks(3.5, 1) == 3.5
    seeds, used = pairqueue.shard_seeds(0, 3)
    assert seeds == used == [0, 1, 2]
    assert pairqueue.job_throughput(3e6, 1.5, 1) == pytest.approx(2.0)
