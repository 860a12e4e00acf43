"""Pre-training, fp64 -- TEST INFRASTRUCTURE ONLY.

The "pre-train" half of the paradigm (§3.1-3.2, App. B-C):

* Alg. 3 table augmentation: every table of the pool at
  every dimension of a set (App. F: {4, 8, 16, 32, 64, 128});
* Alg. 4 random table combinations and the random subset
  of Alg. 5 line 5 are pure random sampling: they live in the seeded input
  generator (workload/pretrain_synth.py), both sides receive the index lists;
* Alg. 5 random table placement: sort by dimension, then per
  table with probability p the memory-feasible device with the lowest device
  dimension, else a uniformly random memory-feasible device -- ``place``;
* labels: the paper measures them on GPUs (PARAM micro-benchmarks);
  no GPU cluster or trace exists here, so the labels come from SPEC.md's
  analytic cost model (its constants S:113) -- ``compute_label``,
  ``comm_labels`` (reading F2-L);
* App. C: the two architectures and the MSE loss, trained
  with Adam, lr 1e-3, other settings default --
  ``compute_loss_grad``, ``comm_loss_grad``, ``adam_step``.  The MSE is the
  mean over the batch (torch.nn.MSELoss default) of the squared error (the
  comm model: mean over batch x D outputs).

Parameter vectors are flat fp64 arrays: for each layer W ([out][in],
row-major, torch.nn.Linear layout) then b, layers in forward order.
"""
from __future__ import annotations

import math
from typing import List, Sequence, Tuple

import numpy as np

from .model import featurize  # noqa: F401  (R1 features of augmented tables)

# SPEC.md:113 OracleParams defaults (invented there; roles from §2 Obs. 1-3)
KAPPA_W = 2.5e-3
OVERHEAD = 0.15
LAUNCH = 0.5
FUSION_GAMMA = 0.3
DIM_EXP = 0.8
HASH_COEF = 0.05
SKEW_COEF = 0.3
COMM_LATENCY = 1.0
BETA = {"fwd": 0.010, "bwd": 0.012}

COMPUTE_WIDTHS = [(5, 128), (128, 32), (32, 64), (64, 1)]   # enc "128-32", head "32-64" + output


def comm_widths(D: int) -> List[Tuple[int, int]]:
    """Comm model "128-64-32-16": 2D -> 128 -> 64 -> 32 -> 16 -> D."""
    w = [2 * D, 128, 64, 32, 16, D]
    return [(w[i], w[i + 1]) for i in range(5)]


def n_params(widths) -> int:
    return sum(i * o + o for i, o in widths)


def unflatten(theta: np.ndarray, widths) -> List[Tuple[np.ndarray, np.ndarray]]:
    out, k = [], 0
    for i, o in widths:
        W = theta[k:k + i * o].reshape(o, i)
        k += i * o
        b = theta[k:k + o]
        k += o
        out.append((W, b))
    return out


def flatten(layers) -> np.ndarray:
    return np.concatenate([np.concatenate([W.ravel(), b]) for W, b in layers])


# ------------------------------------------------------------------ Alg. 3
def augment(dims_of_pool: Sequence[int], dims: Sequence[int]) -> List[Tuple[int, int]]:
    """Alg. 3: for each table, for each dimension in the
    set, the table with that dimension.  Returns (pool table, dim) pairs in
    that loop order."""
    return [(t, int(d)) for t in range(len(dims_of_pool)) for d in dims]


# ------------------------------------------------------------------ labels (SPEC)
def work(dim: int, hash_size: int, pooling: float, skew: float) -> float:
    """kappa_w * pooling * dim^0.8 * (1 + 0.05 log10 hash) *
    (1 - 0.3 min(skew, 2) / 2)."""
    return (KAPPA_W * pooling * dim ** DIM_EXP * (1.0 + HASH_COEF * math.log10(hash_size))
            * (1.0 - SKEW_COEF * min(skew, 2.0) / 2.0))


def compute_label(tables: Sequence[Tuple[int, int, float, float]]) -> float:
    """computation cost of a table combination (dim, hash,
    pooling, skew): launch + sum_t (gamma * overhead + work(t)); a single
    table pays the full overhead (unfused lookup)."""
    if len(tables) == 0:
        raise ValueError("empty combination")
    if len(tables) == 1:
        return LAUNCH + OVERHEAD + work(*tables[0])
    return LAUNCH + sum(FUSION_GAMMA * OVERHEAD + work(*t) for t in tables)


def comm_labels(starts: Sequence[float], devdims: Sequence[float], direction: str) -> np.ndarray:
    """T_end = max_j starts_j + latency + beta_dir * max_j dims_j;
    cost_d = T_end - starts_d (each device's measured latency)."""
    s = np.asarray(starts, np.float64)
    t_end = s.max() + COMM_LATENCY + BETA[direction] * float(np.max(devdims))
    return t_end - s


# ------------------------------------------------------------------ Alg. 5
def place(dims: Sequence[int], sizes: Sequence[int], D: int, cap: int, p: float,
          u: Sequence[float], r: Sequence[float]):
    """Alg. 5 lines 6-16 for one placement.

    dims/sizes: the sampled tables (line 5, in sampling order); p: the greedy
    probability (line 7); u[i], r[i]: the uniforms of the i-th table in the
    sorted order -- p' (line 9) and the random choice (line 13).
    * sort descending by dimension, ties by sampling order (line 6);
    * candidates = devices where the table fits the memory cap (line 10);
      none -> the placement is invalid (reading F2-P);
    * p' <= p: the candidate with the lowest device dimension, lowest index on
      ties (line 12); else candidate number floor(r * |candidates|) in device
      order (line 14).
    Returns (assign per sampled table, device dims, valid)."""
    order = sorted(range(len(dims)), key=lambda i: (-int(dims[i]), i))
    dd = [0] * D
    mem = [0] * D
    assign = [-1] * len(dims)
    for k, i in enumerate(order):
        cand = [d for d in range(D) if mem[d] + int(sizes[i]) <= cap]
        if not cand:
            return assign, dd, False
        if u[k] <= p:
            d = min(cand, key=lambda c: (dd[c], c))
        else:
            d = cand[min(int(math.floor(r[k] * len(cand))), len(cand) - 1)]
        assign[i] = d
        dd[d] += int(dims[i])
        mem[d] += int(sizes[i])
    return assign, dd, True


# ------------------------------------------------------------------ models
def _relu(x):
    return np.maximum(x, 0.0)


def compute_loss_grad(theta: np.ndarray, feats: np.ndarray, sample_off: Sequence[int],
                      labels: np.ndarray):
    """MSE loss and its gradient for the computation cost model (P:219,
    P:688, App. C): per table row e = ReLU(W2 ReLU(W1 x + b1) + b2); per
    sample s = sum of its rows' e; y = H2 ReLU(H1 s + hb1) + hb2;
    L = mean_samples (y - label)^2.  Plain backpropagation, sample by sample."""
    (W1, b1), (W2, b2), (H1, hb1), (H2, hb2) = unflatten(theta, COMPUTE_WIDTHS)
    g = [[np.zeros_like(W), np.zeros_like(b)] for W, b in unflatten(theta, COMPUTE_WIDTHS)]
    B = len(labels)
    loss = 0.0
    for s in range(B):
        rows = range(sample_off[s], sample_off[s + 1])
        z1 = [W1 @ feats[r] + b1 for r in rows]
        h1 = [_relu(z) for z in z1]
        z2 = [W2 @ h + b2 for h in h1]
        e = [_relu(z) for z in z2]
        ssum = np.zeros(32)
        for ei in e:
            ssum = ssum + ei
        za = H1 @ ssum + hb1
        a = _relu(za)
        y = float(H2[0] @ a + hb2[0])
        err = y - float(labels[s])
        loss += err * err / B
        dy = 2.0 * err / B
        g[3][0] += dy * a[None, :]
        g[3][1] += np.array([dy])
        da = dy * H2[0] * (za > 0)
        g[2][0] += np.outer(da, ssum)
        g[2][1] += da
        ds = H1.T @ da
        for k, r in enumerate(rows):
            dz2 = ds * (z2[k] > 0)
            g[1][0] += np.outer(dz2, h1[k])
            g[1][1] += dz2
            dz1 = (W2.T @ dz2) * (z1[k] > 0)
            g[0][0] += np.outer(dz1, feats[r])
            g[0][1] += dz1
    return loss, flatten(g)


def comm_loss_grad(theta: np.ndarray, x: np.ndarray, y: np.ndarray, D: int):
    """MSE loss and gradient for a communication cost model:
    MLP 2D -> 128 -> 64 -> 32 -> 16 -> D, ReLU on hidden layers;
    L = mean over samples and devices of (pred - y)^2."""
    widths = comm_widths(D)
    layers = unflatten(theta, widths)
    g = [[np.zeros_like(W), np.zeros_like(b)] for W, b in layers]
    B = x.shape[0]
    loss = 0.0
    for s in range(B):
        hs, zs = [x[s]], []
        for li, (W, b) in enumerate(layers):
            z = W @ hs[-1] + b
            zs.append(z)
            hs.append(_relu(z) if li < 4 else z)
        err = hs[-1] - y[s]
        loss += float(err @ err) / (B * D)
        dz = 2.0 * err / (B * D)
        for li in range(4, -1, -1):
            W, _ = layers[li]
            g[li][0] += np.outer(dz, hs[li])
            g[li][1] += dz
            if li > 0:
                dz = (W.T @ dz) * (zs[li - 1] > 0)
    return loss, flatten(g)


def adam_step(theta, m, v, grad, t: int, lr: float = 1e-3, b1: float = 0.9, b2: float = 0.999,
              eps: float = 1e-8):
    """torch.optim.Adam (defaults, "learning rate of 0.001 with
    the other configurations as the default"), step t >= 1:
    m = b1 m + (1-b1) g; v = b2 v + (1-b2) g^2;
    theta -= lr * (m / (1 - b1^t)) / (sqrt(v / (1 - b2^t)) + eps)."""
    m = b1 * m + (1.0 - b1) * grad
    v = b2 * v + (1.0 - b2) * grad * grad
    mhat = m / (1.0 - b1 ** t)
    denom = np.sqrt(v / (1.0 - b2 ** t)) + eps
    return theta - lr * mhat / denom, m, v


def pool_features(pool) -> np.ndarray:
    """R1 features of every (augmented) table: [dim, hash, pooling, skew] rows."""
    return np.array([featurize(int(d), int(h), float(p), float(s)) for d, h, p, s in pool])
