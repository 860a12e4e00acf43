"""GPU parity of the fused embedding-bag evaluator (SURVEY §8(f) F3,
k_embag.cu) against oracle/embag.py on the same seeded shard.  fp32 on the
GPU, fp64 in the oracle: each output element is within the fp32 summation
bound n * 2^-24 * sum|x| of the exact sum (n = terms added); each updated
weight within (count + 2) * 2^-24 * (|W| + lr * sum|g|) (lr in fp32, one
rounding per product and per add)."""
import numpy as np
import pytest

from oracle import embag as oe
from workload.pretrain_synth import gen_bag_indices

pytestmark = pytest.mark.gpu
U = 2.0 ** -24


@pytest.fixture(scope="module")
def env():
    import torch
    assert torch.cuda.is_available()
    import paper_2305_01868_b200 as ns
    ctx = ns.ns_create(0)
    yield ns, ctx, torch
    ns.ns_destroy(ctx)


def _shard(B, seed):
    rng = np.random.default_rng(seed)
    # every lane width: dim 4 (1 lane, 32 bags/warp) ... 128 (32 lanes, 1 bag/warp)
    specs = [(1000, 4, 2.0, 0.3), (3000, 8, 5.0, 1.1), (777, 16, 0.5, 0.0), (5000, 32, 12.0, 1.5),
             (20000, 64, 20.0, 0.8), (4096, 128, 7.0, 1.0), (10, 12, 3.0, 0.0)]
    W, I, O = [], [], []
    for rows, dim, pool, skew in specs:
        W.append((rng.normal(size=(rows, dim)) * 0.1).astype(np.float32))
        o, i = gen_bag_indices(rows, pool, skew, B, rng)
        I.append(i)
        O.append(o)
    return W, I, O


def _dev(torch, W, I, O):
    return [(torch.from_numpy(w.copy()).cuda(), torch.from_numpy(i).cuda(), torch.from_numpy(o).cuda())
            for w, i, o in zip(W, I, O)]


@pytest.mark.parametrize("B", [1, 37, 1000])
def test_forward_backward_match_oracle(env, B):
    ns, ctx, torch = env
    W, I, O = _shard(B, seed=B)
    tabs = _dev(torch, W, I, O)
    C = sum(w.shape[1] for w in W)
    out = torch.full((B, C), float("nan"), dtype=torch.float32, device="cuda")
    ns.ns_embedding_bag_forward(ctx, tabs, B, out)
    got = out.cpu().numpy().astype(np.float64)
    ref = oe.bag_forward(W, I, O, B)
    absum = oe.bag_forward([np.abs(w) for w in W], I, O, B)
    n = np.concatenate([np.repeat(np.diff(o)[:, None], w.shape[1], axis=1) for w, o in zip(W, O)], axis=1)
    assert np.all(np.abs(got - ref) <= n * U * absum + 1e-30)
    # backward + SGD
    g = np.random.default_rng(B + 1).normal(size=(B, C)).astype(np.float32)
    lr = 0.01
    ns.ns_embedding_bag_backward_sgd(ctx, tabs, B, torch.from_numpy(g).cuda(), lr)
    new = oe.bag_backward_sgd(W, I, O, g.astype(np.float64), lr)
    gabs = oe.bag_backward_sgd([np.zeros_like(w) for w in W], I, O, -np.abs(g.astype(np.float64)), lr)  # lr*sum|g|
    for t, (w, i, o) in enumerate(zip(W, I, O)):
        cnt = np.bincount(i, minlength=w.shape[0])[:, None]
        # per occurrence: lr rounded to fp32, the product and the add each round once
        bound = (cnt + 2) * U * (np.abs(w) + gabs[t]) + 1e-30
        err = np.abs(tabs[t][0].cpu().numpy().astype(np.float64) - new[t])
        assert np.all(err <= bound), (t, float((err / bound).max()), np.unravel_index(np.argmax(err / bound), err.shape))


def test_bench_shard_sampled(env):
    """The bench's launch shape (batch 65536, C2-style shard) checked on a
    sample of bags against the oracle's definition."""
    ns, ctx, torch = env
    B = 65536
    rng = np.random.default_rng(7)
    specs = [(200_000, 128, 15.0, 1.0), (1_000_000, 64, 30.0, 0.5), (50_000, 16, 5.0, 1.5)]
    tabs, host = [], []
    for rows, dim, pool, skew in specs:
        w = (torch.randn((rows, dim), device="cuda", generator=torch.Generator("cuda").manual_seed(rows)) * 0.1)
        o, i = gen_bag_indices(rows, pool, skew, B, rng)
        tabs.append((w.float(), torch.from_numpy(i).cuda(), torch.from_numpy(o).cuda()))
        host.append((o, i))
    C = sum(d for _, d, _, _ in specs)
    out = torch.zeros((B, C), dtype=torch.float32, device="cuda")
    ns.ns_embedding_bag_forward(ctx, tabs, B, out)
    got = out.cpu().numpy()
    c = 0
    for (w, _, _), (o, i), (_, dim, _, _) in zip(tabs, host, specs):
        for b in range(0, B, 4099):
            rows = torch.from_numpy(i[o[b]:o[b + 1]]).cuda()
            ref = w[rows].double().sum(0).cpu().numpy() if len(rows) else np.zeros(dim)
            bound = len(rows) * U * (w[rows].double().abs().sum(0).cpu().numpy() if len(rows) else 0) + 1e-30
            assert np.all(np.abs(got[b, c:c + dim] - ref) <= bound)
        c += dim


# ------------------------------------------------------------- exchange (F3, multi-GPU half)
def _global_tables(B, seed):
    """Seeded global table set of a DLRM embedding step and its bags (all
    samples of the global batch)."""
    rng = np.random.default_rng(seed)
    specs = [(3000, 16, 4.0, 0.8), (800, 8, 2.0, 0.0), (5000, 32, 6.0, 1.2), (1200, 4, 3.0, 0.5),
             (2500, 64, 5.0, 1.0), (700, 12, 1.0, 0.3)]
    W, I, O = [], [], []
    for rows, dim, pool, skew in specs:
        W.append((rng.normal(size=(rows, dim)) * 0.1).astype(np.float32))
        o, i = gen_bag_indices(rows, pool, skew, B, rng)
        I.append(i)
        O.append(o)
    return W, I, O


def _exchange_check(ns, ctx, torch, world, rank, B=48, seed=11):
    """One rank's forward exchange, backward exchange + SGD on its shard
    (tables t with t % world == rank), against the oracle's global step
    (oracle/embag: bag_forward of every table, exchange_forward, the
    gradient's exchange_backward, bag_backward_sgd).  Returns error strings."""
    W, I, O = _global_tables(B, seed)
    owner = [t % world for t in range(len(W))]
    order = [t for r in range(world) for t in range(len(W)) if owner[t] == r]   # global column order by rank
    cols = [sum(W[t].shape[1] for t in range(len(W)) if owner[t] == r) for r in range(world)]
    Wg, Ig, Og = [W[t] for t in order], [I[t] for t in order], [O[t] for t in order]
    pooled = oe.bag_forward(Wg, Ig, Og, B)
    absum = oe.bag_forward([np.abs(w) for w in Wg], Ig, Og, B)
    n = np.concatenate([np.repeat(np.diff(o)[:, None], w.shape[1], axis=1) for w, o in zip(Wg, Og)], axis=1)
    want = oe.exchange_forward(pooled, cols)[rank]
    bound = oe.exchange_forward(n * U * absum + 1e-30, cols)[rank]
    mine = [t for t in order if owner[t] == rank]
    tabs = _dev(torch, [W[t] for t in mine], [I[t] for t in mine], [O[t] for t in mine])
    out = torch.full((B, cols[rank]), float("nan"), dtype=torch.float32, device="cuda")
    recv = torch.full((len(want),), float("nan"), dtype=torch.float32, device="cuda")
    ns.ns_embedding_bag_forward_exchange(ctx, tabs, B, cols, out, recv)
    errs = []
    got = recv.cpu().numpy().astype(np.float64)
    if not np.all(np.abs(got - want) <= bound):
        errs.append(f"rank {rank}: forward exchange off by {np.max(np.abs(got - want) - bound)}")
    # backward: the global gradient, each rank holding its samples' rank-blocked rows
    g = np.random.default_rng(seed + 1).normal(size=(B, sum(cols))).astype(np.float32)
    grecv = torch.from_numpy(oe.exchange_forward(g.astype(np.float64), cols)[rank].astype(np.float32)).cuda()
    gout = torch.full((B, cols[rank]), float("nan"), dtype=torch.float32, device="cuda")
    lr = 0.02
    ns.ns_embedding_bag_backward_exchange_sgd(ctx, tabs, B, cols, grecv, gout, lr)
    back = oe.exchange_backward(oe.exchange_forward(g.astype(np.float64), cols), cols)[rank]
    if not np.array_equal(gout.cpu().numpy().astype(np.float64), back):
        errs.append(f"rank {rank}: backward exchange differs")
    c0 = sum(cols[:rank])
    new = oe.bag_backward_sgd([W[t] for t in mine], [I[t] for t in mine], [O[t] for t in mine],
                              g[:, c0:c0 + cols[rank]].astype(np.float64), lr)
    gabs = oe.bag_backward_sgd([np.zeros_like(W[t]) for t in mine], [I[t] for t in mine], [O[t] for t in mine],
                               -np.abs(g[:, c0:c0 + cols[rank]].astype(np.float64)), lr)
    for k, t in enumerate(mine):
        cnt = np.bincount(I[t], minlength=W[t].shape[0])[:, None]
        bnd = (cnt + 2) * U * (np.abs(W[t]) + gabs[k]) + 1e-30
        if not np.all(np.abs(tabs[k][0].cpu().numpy().astype(np.float64) - new[k]) <= bnd):
            errs.append(f"rank {rank}: SGD update of table {t} off")
    return errs


def test_exchange_one_rank(env):
    """Without a communicator the exchange is the one-rank copy; with a real
    one-rank NCCL communicator it runs ncclSend/ncclRecv to self."""
    ns, ctx, torch = env
    assert _exchange_check(ns, ctx, torch, 1, 0) == []
    c2 = ns.ns_create(0)
    try:
        ns.ns_comm_init(c2, 1, 0, ns.ns_comm_unique_id())
        assert _exchange_check(ns, c2, torch, 1, 0, B=37, seed=3) == []
    finally:
        ns.ns_destroy(c2)


def _exchange_rank_main(rank, world, port, q):
    import os
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    import paper_2305_01868_b200 as ns
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        ctx = ns.ns_create(0)
        ag, ar = ns.torch_host_comm()
        ns.ns_comm_init_host(ctx, world, rank, ag, ar, ns.torch_host_alltoallv())
        errs = _exchange_check(ns, ctx, torch, world, rank, B=12 * world)
        ns.ns_destroy(ctx)
        dist.destroy_process_group()
        q.put((rank, errs))
    except BaseException as e:   # pragma: no cover
        import traceback
        q.put((rank, [f"exception: {e!r}\n{traceback.format_exc()}"]))


@pytest.mark.parametrize("world", [2, 3])
def test_exchange_multiprocess(world):
    """world processes share GPU 0 (NCCL refuses two ranks on one device) and
    exchange through the host transport: every rank's received pooled rows,
    returned gradients and updated shard equal the oracle's global step."""
    import socket

    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctxm = mp.get_context("spawn")
    q = ctxm.Queue()
    procs = [ctxm.Process(target=_exchange_rank_main, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(res[r] == [] for r in range(world)), res
