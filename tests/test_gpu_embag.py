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
