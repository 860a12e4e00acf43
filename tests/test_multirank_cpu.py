"""World-size-2 gloo test of the bench's multi-rank host logic (CPU): the
job time is the max over ranks, the work is the sum, and weak scaling gives
each rank disjoint tasks."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    t = bench.allreduce_max(world, 10.0 + rank)
    w = bench.allreduce_sum(world, 100.0 * (rank + 1))
    tasks = bench.rank_tasks("C1", 3, rank)
    q.put((rank, t, w, [tk.seed for tk in tasks]))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_aggregation_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    assert all(r[1] == 11.0 for r in res)          # max over ranks
    assert all(r[2] == 300.0 for r in res)         # sum over ranks
    seeds = [set(r[3]) for r in res]
    assert not (seeds[0] & seeds[1])               # disjoint tasks per rank
