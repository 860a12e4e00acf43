"""Pins for oracle/pretrain.py against things other than
itself: torch.autograd and torch.optim.Adam (library routines), central
finite differences, SPEC.md's worked label examples, the
greedy-balance bound and an independently written LPT for Alg. 5 with p = 1.
CPU only."""
import math

import numpy as np
import pytest
import torch

from oracle import pretrain as opt
from workload.pretrain_synth import AUG_DIMS, gen_combinations, gen_placement_draws, gen_pool, init_params


def _compute_batch(seed=0, n=6):
    pool = gen_pool(40, seed=seed + 1)
    aug = opt.augment(pool.dims, AUG_DIMS)
    off, idx = gen_combinations(len(aug), n, 1, 5, seed=seed + 2)
    feats = np.stack([opt.featurize(aug[a][1], int(pool.hash[aug[a][0]]), float(pool.pooling[aug[a][0]]),
                                    float(pool.skew[aug[a][0]])) for a in idx])
    labels = np.array([opt.compute_label([(aug[a][1], int(pool.hash[aug[a][0]]), float(pool.pooling[aug[a][0]]),
                                           float(pool.skew[aug[a][0]])) for a in idx[off[s]:off[s + 1]]])
                       for s in range(n)])
    return feats, off, labels


def _torch_compute_loss(theta, feats, off, labels):
    (W1, b1), (W2, b2), (H1, hb1), (H2, hb2) = opt.unflatten(theta, opt.COMPUTE_WIDTHS)
    X = torch.from_numpy(feats)
    e = torch.relu(torch.relu(X @ W1.T + b1) @ W2.T + b2)
    S = torch.stack([e[off[s]:off[s + 1]].sum(0) for s in range(len(labels))])
    y = (torch.relu(S @ H1.T + hb1) @ H2.T + hb2)[:, 0]
    return torch.nn.functional.mse_loss(y, torch.from_numpy(labels))


def test_compute_grad_matches_autograd():
    feats, off, labels = _compute_batch()
    theta = init_params(opt.COMPUTE_WIDTHS, seed=3)
    loss, grad = opt.compute_loss_grad(theta, feats, off, labels)
    th = torch.tensor(theta, requires_grad=True)
    ref = _torch_compute_loss(th, feats, off, labels)
    ref.backward()
    assert loss == pytest.approx(float(ref), rel=1e-13)
    np.testing.assert_allclose(grad, th.grad.numpy(), rtol=1e-10, atol=1e-13)


def test_comm_grad_matches_autograd():
    D = 4
    rng = np.random.default_rng(5)
    x = rng.uniform(0, 1, (7, 2 * D))
    y = rng.uniform(0, 5, (7, D))
    theta = init_params(opt.comm_widths(D), seed=4)
    loss, grad = opt.comm_loss_grad(theta, x, y, D)
    th = torch.tensor(theta, requires_grad=True)
    h = torch.from_numpy(x)
    for li, (W, b) in enumerate(opt.unflatten(th, opt.comm_widths(D))):
        h = h @ W.T + b
        if li < 4:
            h = torch.relu(h)
    ref = torch.nn.functional.mse_loss(h, torch.from_numpy(y))
    ref.backward()
    assert loss == pytest.approx(float(ref), rel=1e-13)
    np.testing.assert_allclose(grad, th.grad.numpy(), rtol=1e-10, atol=1e-13)


@pytest.mark.parametrize("which", ["compute", "comm"])
def test_gradients_match_central_differences(which):
    rng = np.random.default_rng(11)
    if which == "compute":
        feats, off, labels = _compute_batch(seed=7, n=4)
        theta = init_params(opt.COMPUTE_WIDTHS, seed=8)
        f = lambda t: opt.compute_loss_grad(t, feats, off, labels)   # noqa: E731
    else:
        D = 3
        x, y = rng.uniform(0, 1, (5, 2 * D)), rng.uniform(0, 3, (5, D))
        theta = init_params(opt.comm_widths(D), seed=9)
        f = lambda t: opt.comm_loss_grad(t, x, y, D)   # noqa: E731
    _, g = f(theta)
    for k in rng.choice(len(theta), 25, replace=False):
        h = 1e-6
        tp, tm = theta.copy(), theta.copy()
        tp[k] += h
        tm[k] -= h
        fd = (f(tp)[0] - f(tm)[0]) / (2 * h)
        assert fd == pytest.approx(g[k], rel=1e-5, abs=1e-9), k


def test_adam_matches_torch_optim():
    rng = np.random.default_rng(2)
    theta = rng.normal(size=50)
    th = torch.tensor(theta.copy(), requires_grad=True)
    opt_t = torch.optim.Adam([th], lr=1e-3)     # lr 0.001, other settings default
    m, v = np.zeros(50), np.zeros(50)
    for t in range(1, 6):
        g = rng.normal(size=50) * (10.0 ** rng.integers(-6, 2))
        th.grad = torch.from_numpy(g.copy())
        opt_t.step()
        theta, m, v = opt.adam_step(theta, m, v, g, t)
        np.testing.assert_allclose(theta, th.detach().numpy(), rtol=1e-13, atol=1e-16)


def test_labels_spec_examples():
    # dim 64, pooling 15, hash 1e6, skew 0 -> kappa * 15 * 64^0.8 * 1.3
    assert opt.work(64, 10**6, 15.0, 0.0) == pytest.approx(2.5e-3 * 15 * 64 ** 0.8 * 1.3, rel=1e-15)
    # skew 2 vs 0 -> ratio exactly (1 - skew_coef)
    assert opt.work(32, 10**5, 7.0, 2.0) / opt.work(32, 10**5, 7.0, 0.0) == pytest.approx(0.7, rel=1e-15)
    # one table pays the full overhead; 10 tables: sum of singles
    # - multi = 9 launch + 10 (1 - gamma) overhead
    ts = [(4 * (k + 1), 10 ** (4 + k % 3), 3.0 + k, 0.1 * k) for k in range(10)]
    single = [opt.compute_label([t]) for t in ts]
    assert single[0] == pytest.approx(0.5 + 0.15 + opt.work(*ts[0]), rel=1e-15)
    assert sum(single) - opt.compute_label(ts) == pytest.approx(9 * 0.5 + 10 * 0.7 * 0.15, rel=1e-12)
    # starts 0, dims [100] x 4, fwd -> every device 1.0 + 0.010 * 100 = 2.0 ms
    np.testing.assert_allclose(opt.comm_labels([0, 0, 0, 0], [100] * 4, "fwd"), [2.0] * 4, rtol=1e-15)
    # a device starting 5 ms late measures 5 ms less
    c = opt.comm_labels([0, 5, 0, 0], [100, 50, 80, 10], "bwd")
    assert c[0] - c[1] == pytest.approx(5.0, rel=1e-15) and c[0] == pytest.approx(5 + 1 + 0.012 * 100)


def test_augment_is_the_cross_product():
    # Alg. 3: every table at every dimension, in loop order
    aug = opt.augment([64, 32, 8], AUG_DIMS)
    assert len(aug) == 18 and aug[:6] == [(0, d) for d in AUG_DIMS] and aug[-1] == (2, 128)


def _lpt(dims, D):
    """Textbook LPT on dims: sort descending (stable), each to the least loaded."""
    order = sorted(range(len(dims)), key=lambda i: (-dims[i], i))
    load, a = [0] * D, [-1] * len(dims)
    for i in order:
        d = min(range(D), key=lambda k: (load[k], k))
        a[i] = d
        load[d] += dims[i]
    return a, load


@pytest.mark.parametrize("seed", range(5))
def test_placement_greedy_is_lpt_when_p_is_one(seed):
    # Alg. 5 with p = 1 and no memory pressure is LPT on the dimensions
    # (line 12 "lowest device dimension"); balance bound max - min <= max dim
    rng = np.random.default_rng(seed)
    dims = (4 * rng.integers(1, 33, size=30)).tolist()
    D = 2 + seed % 4
    a, dd, ok = opt.place(dims, [1] * 30, D, 10**12, 1.0, rng.uniform(0, 1, 30), rng.uniform(0, 1, 30))
    ref, load = _lpt(dims, D)
    assert ok and a == ref and dd == load
    assert max(dd) - min(dd) <= max(dims)


def test_placement_random_branch_and_memory():
    # p = 0: table k of the sorted order goes to candidate floor(r_k * |cand|)
    dims, sizes = [8, 16, 4], [10, 10, 10]
    a, dd, ok = opt.place(dims, sizes, 3, 100, 0.0, [0.5, 0.5, 0.5], [0.99, 0.0, 0.5])
    # sorted: 16 (idx1, r=.99 -> cand 2), 8 (idx0, r=0 -> cand 0), 4 (idx2, r=.5 -> cand 1)
    assert ok and a == [0, 2, 1] and dd == [8, 4, 16]
    # memory: the only device with room is forced even when greedy would pick another
    a, dd, ok = opt.place([8, 8], [60, 60], 2, 100, 1.0, [0.0, 0.0], [0.0, 0.0])
    assert ok and a == [0, 1]
    # no feasible device -> invalid placement (reading F2-P)
    _, _, ok = opt.place([8, 8, 8], [60, 60, 60], 2, 100, 1.0, [0.0] * 3, [0.0] * 3)
    assert not ok


def test_placement_coverage_of_balance():
    # §3.1 "p can indirectly control the degree of balance": the draws span
    # balanced (p near 1) and imbalanced (p near 0) plans
    pool = gen_pool(100, seed=3)
    aug = opt.augment(pool.dims, AUG_DIMS)
    dr = gen_placement_draws(len(aug), 300, 4, 10, 60, seed=4)
    ratios = []
    for s in range(300):
        ids = dr.idx[dr.off[s]:dr.off[s + 1]]
        dims = [aug[a][1] for a in ids]
        _, dd, ok = opt.place(dims, [1] * len(dims), 4, 10**12, dr.p[s], dr.u[dr.off[s]:dr.off[s + 1]],
                              dr.r[dr.off[s]:dr.off[s + 1]])
        ratios.append(max(dd) / (sum(dd) / 4))
    assert min(ratios) < 1.05 and max(ratios) > 1.5
