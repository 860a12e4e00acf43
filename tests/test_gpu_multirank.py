"""Multi-rank search with real separate processes.

NCCL refuses two ranks on one GPU and the GPU box has one, so two processes
share GPU 0 and exchange through ns_comm_init_host with torch.distributed
(gloo) callbacks: the same partitioning, allgather of per-trajectory keys,
owner-only assignment rows + int8 allreduce-max and packed-key consistency
check as the NCCL backend.  Every rank's results must equal its own
single-rank run bit for bit.  A one-rank real NCCL communicator
(ns_comm_init with an id) exercises the NCCL calls themselves."""
import os
import socket

import numpy as np
import pytest

from workload.synth import gen_plans, gen_tasks, gen_weights

pytestmark = pytest.mark.gpu

KEYS = ("cost", "n_col", "col_plan", "assign", "grid_index", "n_scores")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _workloads(ns, ctx):
    """(name, callable(ctx) -> dict) of the calls compared across world sizes."""
    w4 = gen_weights(4, "mono")
    w128 = gen_weights(128, "mono")
    t4 = gen_tasks("C2", 7, T=18)
    t5 = gen_tasks("C5", 1, start=3, T=300)
    plans = gen_plans(18, 4, 1000, seed=2)

    def run(w, tasks, fn):
        def f(c):
            ns.ns_load_cost_models(c, w)
            desc, off, caps = ns.table_descs(tasks)
            tabs = ns.ns_featurize_tables(c, desc, off, caps)
            try:
                return fn(c, tabs)
            finally:
                tabs.free()
        return f

    return [
        ("tablewise_grouped", run(w4, t4, lambda c, t: ns.ns_shard_tablewise(c, t, 4, M=11, greedy=1))),
        ("tablewise_lanes", run(w4, t4, lambda c, t: ns.ns_shard_tablewise(c, t, 4, M=11, greedy=2))),
        ("columnwise", run(w4, t4, lambda c, t: ns.ns_shard_columnwise(c, t, 4, N=4, K=3, L=3, M=5))),
        ("columnwise_wide", run(w128, t5, lambda c, t: ns.ns_shard_columnwise(c, t, 128, N=4, K=2, L=2, M=5))),
        ("score_plans", run(w4, t4, lambda c, t: dict(zip(("cost", "best", "best_cost"),
                                                         ns.ns_score_plans(c, t, 0, 4, [], plans))))),
    ]


def _same(a, b):
    for k in a:
        if isinstance(a[k], np.ndarray) or k in KEYS or k in ("best", "best_cost"):
            if not np.array_equal(np.asarray(a[k]), np.asarray(b[k])):
                return k
    return None


def _rank_main(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    import paper_2305_01868_b200 as ns
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        ctx = ns.ns_create(0)
        wl = _workloads(ns, ctx)
        ref = {name: f(ctx) for name, f in wl}
        ag, ar = ns.torch_host_comm()
        ns.ns_comm_init_host(ctx, world, rank, ag, ar)
        bad = []
        for name, f in wl:
            got = f(ctx)
            k = _same(ref[name], got) if name != "score_plans" else None
            if name == "score_plans":
                # cost_out holds only this rank's slice; the argmin is global
                if got["best"] != ref[name]["best"] or got["best_cost"] != ref[name]["best_cost"]:
                    k = "best"
                per = (1000 + world - 1) // world
                lo, hi = rank * per, min(1000, (rank + 1) * per)
                if not np.array_equal(got["cost"][lo:hi], ref[name]["cost"][lo:hi]):
                    k = "cost slice"
            if k:
                bad.append(f"{name}:{k}")
        ns.ns_destroy(ctx)
        dist.destroy_process_group()
        q.put((rank, bad))
    except BaseException as e:   # pragma: no cover
        import traceback
        q.put((rank, [f"exception: {e!r}\n{traceback.format_exc()}"]))


@pytest.mark.parametrize("world", [2, 3])
def test_multiprocess_host_comm_matches_single_rank(world):
    import torch.multiprocessing as mp
    ctxm = mp.get_context("spawn")
    q = ctxm.Queue()
    port = _free_port()
    procs = [ctxm.Process(target=_rank_main, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(res[r] == [] for r in range(world)), res


def test_one_rank_real_nccl_communicator():
    """ns_comm_init(nranks=1, id) creates a real NCCL communicator: the
    searches run their collectives through NCCL (allgather of the keys,
    int8 allreduce-max of the winner's row, the consistency allreduce-min)
    and return exactly the plain single-GPU results."""
    import torch
    import paper_2305_01868_b200 as ns
    assert torch.cuda.is_available()
    ctx = ns.ns_create(0)
    try:
        wl = _workloads(ns, ctx)
        ref = {name: f(ctx) for name, f in wl}
        ns.ns_comm_init(ctx, 1, 0, ns.ns_comm_unique_id())
        for name, f in wl:
            got = f(ctx)
            assert _same(ref[name], got) is None, name
    finally:
        ns.ns_destroy(ctx)
