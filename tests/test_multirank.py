"""The N>1 plumbing of bench.py on CPU (gloo, world_size 2), through bench.py's
own functions: the headline's weak-scaling seed shards (disjoint, covering the
master list, each rank's 10-seed sections a prefix of its own shard), the
cfg5 strong-scaling split, the max-over-ranks timing reduction and the
aggregate value, and the `--gpus` / WORLD_SIZE contract."""
import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    master = np.arange(5000, 5000 + bench.SEEDS_PER_RANK * world, dtype=np.uint64)
    shard = bench.seed_shard(master, rank, world, bench.SEEDS_PER_RANK)
    _, ks, ns = bench.SCHEDULE["cfg4"]
    sections = [shard[:n].tolist() for n in ns]
    c5 = bench.cfg5_shard(np.arange(65536, dtype=np.uint64), rank, world)
    # rank-local device times; the job time is the max over ranks
    tmax = bench.max_over_ranks(torch, dist, 10.0 + 5.0 * rank)
    esum = bench.sum_over_ranks(torch, dist, 100.0 * (rank + 1))
    cfg = bench.workload_config("cfg4", world, 7, 9)
    out[rank] = (shard.tolist(), sections, c5.tolist(), tmax, esum, cfg)
    dist.destroy_process_group()


def test_two_rank_bench_plumbing():
    world = 2
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    import bench
    shards = [res[r][0] for r in range(world)]
    assert set(shards[0]).isdisjoint(shards[1])
    assert sorted(shards[0] + shards[1]) == list(range(5000, 5000 + bench.SEEDS_PER_RANK * world))
    for r in range(world):  # the 300/300/10/10 sections are prefixes of the rank's own shard
        secs = res[r][1]
        assert [len(s) for s in secs] == [300, 300, 10, 10]
        assert all(s == shards[r][:len(s)] for s in secs)
    c5 = [res[r][2] for r in range(world)]
    assert c5[0] + c5[1] == list(range(65536)) and len(c5[0]) == 32768 and len(c5[0]) % 64 == 0
    assert all(res[r][3] == 15.0 for r in range(world))       # max over ranks
    assert all(res[r][4] == 300.0 for r in range(world))      # sum over ranks
    assert res[0][5] == res[1][5] and res[0][5]["ranks"] == 2  # one config for the whole job


def test_cfg5_shard_uneven():
    import bench
    m = np.arange(65536)
    parts = [bench.cfg5_shard(m, r, 3) for r in range(3)]
    assert np.array_equal(np.concatenate(parts), m)
    assert max(map(len, parts)) - min(map(len, parts)) <= 1


def test_gpus_flag_must_match_world_size():
    env = dict(os.environ, WORLD_SIZE="3", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2"], env=env,
                       capture_output=True, text=True, timeout=120)
    assert r.returncode != 0 and "--gpus 2 but WORLD_SIZE=3" in r.stderr
