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


def _comm_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import numpy as np
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2305_01868_b200._native import NS_COMM_MAX_I8, NS_COMM_MIN_U64, torch_host_comm
    ag, ar = torch_host_comm()
    send = np.arange(5, dtype=np.uint8) + 10 * rank
    recv = np.zeros(5 * world, np.uint8)
    ag(send, recv)
    # uint64 minimum across the sign bit (order-preserving cost keys live there)
    keys = np.array([0xFFFF000000000000 - rank, 5 + rank, 0x8000000000000000 + rank], dtype=np.uint64)
    ar(keys, NS_COMM_MIN_U64)
    # int8 maximum: the owner's row wins over the others' -128 filler
    row = np.array([-128, -128, -1], np.int8) if rank else np.array([3, 0, -1], np.int8)
    ar(row, NS_COMM_MAX_I8)
    q.put((rank, recv.tolist(), keys.tolist(), row.tolist()))
    dist.barrier()
    dist.destroy_process_group()


def test_host_comm_callbacks_world2():
    """The torch.distributed (gloo) callbacks behind ns_comm_init_host: the
    allgather concatenates in rank order, the uint64 min is unsigned (keys
    above 2^63 are the common case), the int8 max fills in the owner's row."""
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_comm_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict((r, rest) for r, *rest in (q.get(timeout=120) for _ in range(world)))
    for p in ps:
        p.join(timeout=60)
    for r in range(world):
        recv, keys, row = res[r]
        assert recv == [0, 1, 2, 3, 4, 10, 11, 12, 13, 14]
        assert keys == [0xFFFF000000000000 - 1, 5, 0x8000000000000000]
        assert row == [3, 0, -1]


def _a2a_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import numpy as np
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import embag as oe
    from paper_2305_01868_b200._native import torch_host_alltoallv
    # the embedding exchange's host transport on the layouts the library
    # uses: this rank's [B][cols[rank]] pooled rows as nranks sample blocks
    cols, B = [3, 1, 2][:world], 6
    X = np.arange(B * sum(cols), dtype=np.float32).reshape(B, sum(cols))   # the global pooled matrix
    c0 = sum(cols[:rank])
    mine = np.ascontiguousarray(X[:, c0:c0 + cols[rank]])
    Bl = B // world
    send_b = [Bl * cols[rank] * 4] * world
    recv_b = [Bl * c * 4 for c in cols]
    recv = np.zeros(sum(recv_b), np.uint8)
    torch_host_alltoallv()(mine.view(np.uint8).reshape(-1), send_b, recv, recv_b)
    got = recv.view(np.float32)
    ok = np.array_equal(got, oe.exchange_forward(X.astype(np.float64), cols)[rank])
    q.put((rank, bool(ok)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_host_alltoallv_callback_gloo(world):
    """The torch.distributed (gloo) all-to-all callback behind the embedding
    exchange (ns_host_comm.alltoallv): per-peer block sizes differ, the self
    block is copied, and every rank ends with the oracle's rank-blocked
    receive buffer (oracle/embag.exchange_forward)."""
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_a2a_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
    assert all(res[r] for r in range(world)), res
