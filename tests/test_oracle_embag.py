"""Pins for oracle/embag.py against the library routine
torch.nn.functional.embedding_bag (sum mode) and its autograd + SGD, plus
the special cases (single-row bags copy the row, empty bags are zero).  CPU."""
import numpy as np
import torch

from oracle import embag as oe
from workload.pretrain_synth import gen_bag_indices


def _shard(seed=0, B=40):
    rng = np.random.default_rng(seed)
    specs = [(97, 8, 3.0, 0.0), (500, 16, 6.0, 1.2), (64, 4, 1.0, 1.0), (1000, 32, 9.0, 0.6)]
    W, I, O = [], [], []
    for rows, dim, pool, skew in specs:
        W.append(rng.normal(size=(rows, dim)).astype(np.float32))
        o, i = gen_bag_indices(rows, pool, skew, B, rng)
        I.append(i)
        O.append(o)
    return W, I, O, B


def test_forward_matches_torch_embedding_bag():
    W, I, O, B = _shard()
    out = oe.bag_forward(W, I, O, B)
    ref = torch.cat([torch.nn.functional.embedding_bag(torch.from_numpy(i), torch.from_numpy(w).double(),
                                                       torch.from_numpy(o[:-1].astype(np.int64)), mode="sum")
                     for w, i, o in zip(W, I, O)], dim=1)
    np.testing.assert_allclose(out, ref.numpy(), rtol=1e-13, atol=1e-13)


def test_backward_sgd_matches_autograd_sgd():
    W, I, O, B = _shard(seed=3)
    rng = np.random.default_rng(4)
    g = rng.normal(size=(B, sum(w.shape[1] for w in W)))
    lr = 0.05
    new = oe.bag_backward_sgd(W, I, O, g, lr)
    c = 0
    for t, (w, i, o) in enumerate(zip(W, I, O)):
        p = torch.tensor(w.astype(np.float64), requires_grad=True)
        y = torch.nn.functional.embedding_bag(torch.from_numpy(i), p, torch.from_numpy(o[:-1].astype(np.int64)),
                                              mode="sum")
        (y * torch.from_numpy(g[:, c:c + w.shape[1]])).sum().backward()
        opt = torch.optim.SGD([p], lr=lr)
        opt.step()
        np.testing.assert_allclose(new[t], p.detach().numpy(), rtol=1e-13, atol=1e-13)
        c += w.shape[1]


def test_special_cases():
    W = [np.arange(12, dtype=np.float32).reshape(3, 4)]
    off = [np.array([0, 1, 1, 3], np.int32)]           # bag 0: one row, bag 1: empty, bag 2: two rows
    idx = [np.array([2, 0, 2], np.int64)]
    out = oe.bag_forward(W, idx, off, 3)
    assert out[0].tolist() == [8, 9, 10, 11] and out[1].tolist() == [0, 0, 0, 0]
    assert out[2].tolist() == [8, 10, 12, 14]
    new = oe.bag_backward_sgd(W, idx, off, np.ones((3, 4)), 1.0)[0]
    assert new[2].tolist() == [6, 7, 8, 9] and new[0].tolist() == [-1, 0, 1, 2] and new[1].tolist() == [4, 5, 6, 7]


def test_zipf_indices_in_range_and_skewed():
    rng = np.random.default_rng(5)
    o, i = gen_bag_indices(10_000, 20.0, 1.2, 2000, rng)
    assert i.min() >= 0 and i.max() < 10_000 and o[-1] == len(i)
    _, counts = np.unique(i, return_counts=True)
    assert counts.max() > 50 * np.median(counts)       # hot rows exist (skew > 0)
    o, i = gen_bag_indices(10_000, 20.0, 0.0, 2000, rng)
    _, counts = np.unique(i, return_counts=True)
    assert counts.max() < 30                            # skew 0: near uniform


# ------------------------------------------------------------- the exchanges
def test_exchange_hand_example():
    """B = 4 samples, R = 2 ranks, rank 0 owns 1 column, rank 1 two
    (PAPER.md:49): rank 0 receives rows 0-1 of every rank's columns, rank 1
    rows 2-3, each rank-blocked.  Expected values written out by hand."""
    pooled = np.arange(12, dtype=np.float64).reshape(4, 3)
    r0, r1 = oe.exchange_forward(pooled, [1, 2])
    assert r0.tolist() == [0, 3, 1, 2, 4, 5]
    assert r1.tolist() == [6, 9, 7, 8, 10, 11]
    g0, g1 = oe.exchange_backward([r0, r1], [1, 2])
    assert g0.tolist() == [[0], [3], [6], [9]]
    assert g1.tolist() == [[1, 2], [4, 5], [7, 8], [10, 11]]


def test_exchange_elementwise_and_round_trip():
    """Every received element is the pooled element its (rank, block, row,
    column) names (an index loop written independently of the slicing), and
    the backward exchange inverts the forward one (zero-width ranks too)."""
    rng = np.random.default_rng(5)
    for cols, B in (([5, 0, 7], 9), ([3], 4), ([2, 2, 2, 2], 8)):
        R = len(cols)
        X = rng.normal(size=(B, sum(cols)))
        recv = oe.exchange_forward(X, cols)
        Bl = B // R
        for q in range(R):
            pos = 0
            for r in range(R):
                c0 = sum(cols[:r])
                for i in range(Bl):
                    for j in range(cols[r]):
                        assert recv[q][pos] == X[q * Bl + i, c0 + j]
                        pos += 1
            assert pos == len(recv[q])
        back = oe.exchange_backward(recv, cols)
        for r in range(R):
            np.testing.assert_array_equal(back[r], X[:, sum(cols[:r]):sum(cols[:r]) + cols[r]])
    # one rank: the exchange is the identity
    X = rng.normal(size=(6, 4))
    np.testing.assert_array_equal(oe.exchange_forward(X, [4])[0], X.reshape(-1))
