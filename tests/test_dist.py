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
    # the Batch IDA* leg: rank 0 alone drives every GPU (one evaluator each)
    plan = bench.search_plan(r, w)
    cmd = None
    if plan:
        cmd = bench.search_command(plan["impl"], "/tmp/m.bmlp", 0.5, 10, 16, plan["gpus"], plan["evaluators"],
                                   16384, 25, bench.SEARCH_WALK)
    q.put((rank, mx, bench.whole_job_rate(512, 3, w, mx), packed.tobytes(), plan, cmd))
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
    assert res[0][4] == {"impl": "fast", "gpus": 2, "evaluators": 2} and res[1][4] is None
    cmd = res[0][5]
    assert cmd[0].endswith("tools/bin/bida_search_fast")
    assert cmd[cmd.index("--gpus") + 1] == "2" and cmd[cmd.index("--evaluators") + 1] == "2"
    assert cmd[cmd.index("--table1-pdb") + 1] == "8" and "--gpu-pdb" in cmd


def test_single_rank_rate():
    import bench

    assert bench.whole_job_rate(1000, 10, 1, 1000.0) == 10000.0
