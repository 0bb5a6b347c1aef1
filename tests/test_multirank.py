"""The N>1 plumbing of bench.py on CPU (gloo, world_size 2): seed shards are
disjoint and cover the master list; the timing reduction is a max over ranks;
the rank-0 broadcast of the graph arrays reproduces them on every rank."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    master = np.arange(1000, 1000 + 7 * world, dtype=np.uint64)
    shard = bench.seed_shard(master, rank, world, 7)
    # rank-local "device time"; the job time is the max over ranks
    t = torch.tensor([1.0 + rank], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    # graph broadcast from rank 0 (the bench does this over NCCL)
    arr = torch.arange(10, dtype=torch.int32) * 3 if rank == 0 else torch.zeros(10, dtype=torch.int32)
    dist.broadcast(arr, 0)
    out[rank] = (shard.tolist(), float(t[0]), arr.tolist())
    dist.destroy_process_group()


def test_two_rank_shards_and_reductions():
    world = 2
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    shards = [res[r][0] for r in range(world)]
    assert set(shards[0]).isdisjoint(shards[1])
    assert sorted(shards[0] + shards[1]) == list(range(1000, 1000 + 7 * world))
    assert all(res[r][1] == 2.0 for r in range(world))
    assert all(res[r][2] == [3 * i for i in range(10)] for r in range(world))
