"""CPU, world_size 2 over gloo: the multi-GPU bench plumbing (one process per
device, no data-path collective; barrier + max-over-ranks timing) and the
per-rank sharding of synthetic batches."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank), BIDA_BENCH_BACKEND="gloo")
    import bench
    import paper_2507_11916_b200 as bida

    r, w, local = bench.dist_init()
    assert (r, w, local) == (rank, world, rank)
    # each rank times its own shard; the job time is the slowest rank's
    my_ms = 10.0 * (rank + 1)
    mx = bench.reduce_max(my_ms, w)
    bench.barrier(w)
    # per-rank synthetic batches are independent shards (seeded by rank)
    packed = bida.random_walks("rc", 512, 0, 30, seed=1000 * rank)
    q.put((rank, mx, bench.whole_job_rate(512, 3, w, mx), packed.tobytes()))
    import torch.distributed as dist

    dist.destroy_process_group()


def test_two_rank_gloo_bench_plumbing():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    [p.start() for p in procs]
    res = [q.get(timeout=120) for _ in range(2)]
    [p.join(60) for p in procs]
    assert all(p.exitcode == 0 for p in procs)
    res.sort()
    assert res[0][1] == res[1][1] == 20.0          # max over ranks
    assert res[0][2] == res[1][2] == 512 * 3 * 2 / 0.020
    assert res[0][3] != res[1][3]                    # disjoint shards


def test_single_rank_rate():
    import bench

    assert bench.whole_job_rate(1000, 10, 1, 1000.0) == 10000.0
