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
    seeds = pairqueue.shard_seeds(info.rank, world, 7)
    # per-rank "device time": rank 1 is the slow one
    t = 1.0 + rank
    pairqueue.barrier(world)
    tmax = pairqueue.max_over_ranks(t, world)
    # everyone can gather the shards to check disjointness
    gathered = [None] * world
    dist.all_gather_object(gathered, seeds)
    # whole-job throughput: work summed over ranks (rank 1 did less)
    out[rank] = (seeds, pairqueue.weak_seeds(rank, 3), tmax, gathered,
                 pairqueue.job_throughput(len(seeds) * 1e6, tmax, world))
    dist.destroy_process_group()


def test_two_rank_pair_queue_gloo():
    world = 2
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    s0, w0, t0, g0, v0 = res[0]
    s1, w1, t1, g1, v1 = res[1]
    assert s0 == [0, 2, 4, 6] and s1 == [1, 3, 5]     # strong scaling: seeds i::N
    assert not set(s0) & set(s1)                      # disjoint pair queues
    assert sorted(s0 + s1) == list(range(7))          # covering the job once
    assert w0 == [0, 1, 2] and w1 == [3, 4, 5]        # weak scaling (extra mode)
    assert t0 == t1 == 2.0                            # max over ranks
    assert g0 == g1 == [s0, s1]
    assert v0 == v1 == pytest.approx(7e6 / 2.0 / 1e6)  # summed work / max time


def test_single_rank_defaults():
    info = pairqueue.rank_info({})
    assert (info.rank, info.world, info.local) == (0, 1, 0)
    assert pairqueue.max_over_ranks(3.5, 1) == 3.5
    assert pairqueue.shard_seeds(0, 1, 3) == [0, 1, 2]
    assert pairqueue.job_throughput(3e6, 1.5, 1) == pytest.approx(2.0)
    with pytest.raises(ValueError):
        pairqueue.shard_seeds(2, 2, 64)


def _bench_line(*args):
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items()
           if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), *args],
                         capture_output=True, text=True, timeout=600, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout  # rank 0 alone prints
    return json.loads(lines[0])


def test_bench_launcher_two_ranks_dry_run():
    """`bench.py --gpus 2` (no torchrun environment) re-launches itself as two
    ranks; config 4's 64 pairs are sharded i::2 (strong scaling), disjoint,
    covering seeds 0..63 once; time is the max over ranks (gloo here)."""
    d = _bench_line("--gpus", "2", "--dry-run")
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["global_pairs"] == 64
    a, b = d["seeds_by_rank"]
    assert a == list(range(0, 64, 2)) and b == list(range(1, 64, 2))
    assert d["max_time"] == 2.0
    # a single-pair workload does not shard: one replica per rank
    d = _bench_line("--gpus", "2", "--dry-run", "--workload", "c2")
    assert d["scaling"] == "weak" and d["seeds_by_rank"] == [[0], [0]]
    # weak scaling is an explicit extra mode
    d = _bench_line("--gpus", "2", "--dry-run", "--weak", "--pairs", "3")
    assert d["seeds_by_rank"] == [[0, 1, 2], [3, 4, 5]] and d["global_pairs"] == 6
