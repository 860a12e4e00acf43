"""GPU parity of the pre-training path (k_pretrain.cu)
against the fp64 oracle (oracle/pretrain.py) on the same seeded draws:
features and labels of Alg. 4 combinations (1e-13 / 1e-12 relative),
Alg. 5 placements (assignments and validity exact; inputs and labels 1e-13),
and Adam steps of both cost models (loss and every weight after 3 steps
within 1e-11: fp64 on both sides, only the gradient summation order
differs)."""
import numpy as np
import pytest

from oracle import pretrain as opt
from workload.pretrain_synth import AUG_DIMS, gen_combinations, gen_placement_draws, gen_pool, init_params

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch
    assert torch.cuda.is_available()
    import paper_2305_01868_b200 as ns
    ctx = ns.ns_create(0)
    yield ns, ctx, torch
    ns.ns_destroy(ctx)


def _pool_dev(ns, torch, pool):
    desc = np.zeros(pool.n, dtype=ns.TABLE_DESC)
    desc["dim"], desc["hash_size"], desc["pooling_factor"], desc["skew"] = pool.dims, pool.hash, pool.pooling, pool.skew
    return (torch.from_numpy(desc.view(np.uint8)).cuda(),
            torch.tensor(AUG_DIMS, dtype=torch.int32, device="cuda"))


def _aug_table(pool, a):
    t, d = divmod(int(a), len(AUG_DIMS))
    return (AUG_DIMS[d], int(pool.hash[t]), float(pool.pooling[t]), float(pool.skew[t]))


def _compute_data(ns, ctx, torch, n, seed=1):
    pool = gen_pool(120, seed=seed)
    pd, ad = _pool_dev(ns, torch, pool)
    off, idx = gen_combinations(pool.n * len(AUG_DIMS), n, 1, 15, seed=seed + 1)
    off_d, idx_d = torch.from_numpy(off).cuda(), torch.from_numpy(idx).cuda()
    feats = torch.zeros((len(idx), 5), dtype=torch.float64, device="cuda")
    labels = torch.zeros(n, dtype=torch.float64, device="cuda")
    ns.ns_pretrain_compute_samples(ctx, pd, ad, off_d, idx_d, feats, labels)
    torch.cuda.synchronize()
    return pool, off, idx, off_d, feats, labels


def test_compute_samples_match_oracle(env):
    ns, ctx, torch = env
    pool, off, idx, _, feats, labels = _compute_data(ns, ctx, torch, 400)
    F, Y = feats.cpu().numpy(), labels.cpu().numpy()
    for s in range(400):
        tabs = [_aug_table(pool, a) for a in idx[off[s]:off[s + 1]]]
        assert Y[s] == pytest.approx(opt.compute_label(tabs), rel=1e-12, abs=0)
        for k, t in enumerate(tabs):
            np.testing.assert_allclose(F[off[s] + k], opt.featurize(*t), rtol=1e-15, atol=0)


@pytest.mark.parametrize("D,cap", [(4, 4 << 30), (8, 1 << 30)])
def test_comm_samples_match_oracle(env, D, cap):
    ns, ctx, torch = env
    pool = gen_pool(200, seed=5)
    pd, ad = _pool_dev(ns, torch, pool)
    n = 300
    dr = gen_placement_draws(pool.n * len(AUG_DIMS), n, D, 10 * D // 4, 60 * D // 4, seed=6)
    t = lambda a, dt=None: torch.from_numpy(np.ascontiguousarray(a)).cuda()   # noqa: E731
    rows = int(dr.off[-1])
    x = torch.zeros((n, 2 * D), dtype=torch.float64, device="cuda")
    yf, yb = torch.zeros((n, D), dtype=torch.float64, device="cuda"), torch.zeros((n, D), dtype=torch.float64,
                                                                                   device="cuda")
    asg = torch.full((rows,), -1, dtype=torch.int8, device="cuda")
    valid = torch.zeros(n, dtype=torch.uint8, device="cuda")
    ns.ns_pretrain_comm_samples(ctx, pd, ad, D, cap, t(dr.off), t(dr.idx), t(dr.p), t(dr.u), t(dr.r), t(dr.starts),
                                x, yf, yb, asg, valid)
    X, YF, YB, A, V = (a.cpu().numpy() for a in (x, yf, yb, asg, valid))
    n_invalid = 0
    for s in range(n):
        sl = slice(dr.off[s], dr.off[s + 1])
        tabs = [_aug_table(pool, a) for a in dr.idx[sl]]
        dims = [tb[0] for tb in tabs]
        sizes = [tb[1] * tb[0] * 4 for tb in tabs]
        a, dd, ok = opt.place(dims, sizes, D, cap, dr.p[s], dr.u[sl], dr.r[sl])
        assert bool(V[s]) == ok, s
        assert A[sl].tolist() == a, s
        if not ok:
            n_invalid += 1
            continue
        np.testing.assert_allclose(X[s], np.concatenate([dr.starts[s] / 20.0, np.array(dd) / 1024.0]),
                                   rtol=1e-15, atol=0)
        np.testing.assert_allclose(YF[s], opt.comm_labels(dr.starts[s], dd, "fwd"), rtol=1e-13)
        np.testing.assert_allclose(YB[s], opt.comm_labels(dr.starts[s], dd, "bwd"), rtol=1e-13)
    # 4 GiB / D = 4: mostly valid plans; 1 GiB / D = 8: mostly the no-candidate path
    assert 0 < n - n_invalid and (n_invalid < n // 2) == (cap > 1 << 30)


def test_compute_model_adam_steps_match_oracle(env):
    ns, ctx, torch = env
    n, B = 600, 512
    pool, off, idx, off_d, feats, labels = _compute_data(ns, ctx, torch, n, seed=11)
    F, Y = feats.cpu().numpy(), labels.cpu().numpy()
    theta0 = init_params(opt.COMPUTE_WIDTHS, seed=12)
    th = torch.from_numpy(theta0.copy()).cuda()
    m, v = torch.zeros_like(th), torch.zeros_like(th)
    loss = torch.zeros(1, dtype=torch.float64, device="cuda")
    rng = np.random.default_rng(13)
    th_o, m_o, v_o = theta0.copy(), np.zeros_like(theta0), np.zeros_like(theta0)
    maxrows = int(np.max(np.diff(off)))
    for t in range(1, 4):
        batch = rng.permutation(n)[:B].astype(np.int32)
        ns.ns_pretrain_compute_step(ctx, th, m, v, t, 1e-3, feats, off_d, labels, torch.from_numpy(batch).cuda(),
                                    maxrows, loss)
        # oracle on the same batch: rows of the selected samples in batch order
        boff = np.zeros(B + 1, np.int64)
        boff[1:] = np.cumsum([off[s + 1] - off[s] for s in batch])
        bf = np.concatenate([F[off[s]:off[s + 1]] for s in batch])
        lo, g = opt.compute_loss_grad(th_o, bf, boff, Y[batch])
        th_o, m_o, v_o = opt.adam_step(th_o, m_o, v_o, g, t)
        assert float(loss.item()) == pytest.approx(lo, rel=1e-11)
        np.testing.assert_allclose(th.cpu().numpy(), th_o, rtol=0, atol=1e-11)


@pytest.mark.parametrize("D", [4, 8])
def test_comm_model_adam_steps_match_oracle(env, D):
    ns, ctx, torch = env
    rng = np.random.default_rng(20 + D)
    n, B = 700, 512
    Xh = rng.uniform(0, 1, (n, 2 * D))
    Yh = rng.uniform(0, 6, (n, D))
    x, y = torch.from_numpy(Xh).cuda(), torch.from_numpy(Yh).cuda()
    theta0 = init_params(opt.comm_widths(D), seed=21)
    th = torch.from_numpy(theta0.copy()).cuda()
    m, v = torch.zeros_like(th), torch.zeros_like(th)
    loss = torch.zeros(1, dtype=torch.float64, device="cuda")
    th_o, m_o, v_o = theta0.copy(), np.zeros_like(theta0), np.zeros_like(theta0)
    for t in range(1, 4):
        batch = rng.permutation(n)[:B].astype(np.int32)
        ns.ns_pretrain_comm_step(ctx, D, th, m, v, t, 1e-3, x, y, torch.from_numpy(batch).cuda(), loss)
        lo, g = opt.comm_loss_grad(th_o, Xh[batch], Yh[batch], D)
        th_o, m_o, v_o = opt.adam_step(th_o, m_o, v_o, g, t)
        assert float(loss.item()) == pytest.approx(lo, rel=1e-11)
        np.testing.assert_allclose(th.cpu().numpy(), th_o, rtol=0, atol=1e-11)


def test_training_reduces_loss_and_weights_load(env):
    """Pre-train then search: 300 Adam steps lower the compute model's MSE on
    its labels by 10x, and the trained fp64 weights load into the search
    (ns_load_cost_models) unchanged (synthetic-fit weights)."""
    ns, ctx, torch = env
    n, B = 4096, 512
    pool, off, idx, off_d, feats, labels = _compute_data(ns, ctx, torch, n, seed=31)
    th = torch.from_numpy(init_params(opt.COMPUTE_WIDTHS, seed=32)).cuda()
    m, v = torch.zeros_like(th), torch.zeros_like(th)
    loss = torch.zeros(1, dtype=torch.float64, device="cuda")
    rng = np.random.default_rng(33)
    maxrows = int(np.max(np.diff(off)))
    losses = []
    for t in range(1, 301):
        batch = torch.from_numpy(rng.permutation(n)[:B].astype(np.int32)).cuda()
        ns.ns_pretrain_compute_step(ctx, th, m, v, t, 1e-3, feats, off_d, labels, batch, maxrows, loss)
        if t in (1, 300):
            losses.append(float(loss.item()))
    assert losses[1] < 0.1 * losses[0], losses
    # the trained model drives a search: load it with random-init comm models
    import dataclasses
    from workload.synth import gen_tasks, gen_weights
    layers = opt.unflatten(th.cpu().numpy(), opt.COMPUTE_WIDTHS)
    w = dataclasses.replace(gen_weights(4, "mono"), enc=layers[:2], head=layers[2:], kind="pretrained")
    ns.ns_load_cost_models(ctx, w)
    tasks = gen_tasks("C2", 4, T=20)
    desc, off2, caps = ns.table_descs(tasks)
    tabs = ns.ns_featurize_tables(ctx, desc, off2, caps)
    out = ns.ns_shard_tablewise(ctx, tabs, 4, M=11)
    tabs.free()
    from oracle import model as om, search as osr
    for i, task in enumerate(tasks):
        r = osr.greedy_grid_search(w, om.TableEmbeddings(w, task), task, [], 11)
        assert abs(out["cost"][i] - r.cost) <= 1e-12 * abs(r.cost)
