"""Cost models and the plan-cost simulator, fp64 -- TEST INFRASTRUCTURE ONLY.

Follows PAPER.md §3.2 (lines 215-219), App. C (line 688) and §3.3 (line 232),
with the readings of DESIGN.md §"Readings" (R1-R4, R10, R11).
"""
from __future__ import annotations

from typing import Dict, Iterable, List, Sequence, Tuple

import numpy as np

F = 5  # R1: [dim, hash size, pooling factor, indices distribution (skew), size]


def featurize(dim: int, hash_size: int, pooling: float, skew: float) -> np.ndarray:
    """O1.  PAPER.md:111 / :219 list the table factors "dimension, hash size,
    pooling factor, and indices distribution"; BASELINE.json adds size.
    Normalisation constants per SPEC.md:252 (reading R1):
    x = [dim/128, log10(hash)/8, pooling/50, skew/2, hash*dim*4 / 2^30].
    """
    return np.array([
        dim / 128.0,
        np.log10(float(hash_size)) / 8.0,
        float(pooling) / 50.0,
        float(skew) / 2.0,
        float(hash_size) * float(dim) * 4.0 / float(1 << 30),
    ], dtype=np.float64)


def relu(x: np.ndarray) -> np.ndarray:
    return np.maximum(x, 0.0)


def mlp(layers: Sequence[Tuple[np.ndarray, np.ndarray]], x: np.ndarray,
        relu_last: bool) -> np.ndarray:
    """Plain MLP: x <- W x + b layer by layer, ReLU on every hidden layer
    (reading R2), and on the last layer only if ``relu_last``."""
    h = np.asarray(x, dtype=np.float64)
    n = len(layers)
    for i, (W, b) in enumerate(layers):
        h = W @ h + b
        if i < n - 1 or relu_last:
            h = relu(h)
    return h


def encode(weights, x: np.ndarray) -> np.ndarray:
    """O2.  Shared table MLP "128-32", ReLU after both layers
    (reading R2): e = ReLU(W2 ReLU(W1 x + b1) + b2), 5 -> 128 -> 32."""
    return mlp(weights.enc, x, relu_last=True)


def head(weights, s: np.ndarray) -> float:
    """O3.  Head MLP "32-64" then a scalar output:
    h(s) = H2 ReLU(H1 s + hb1) + hb2.  No output clamp (reading R3)."""
    return float(mlp(weights.head, s, relu_last=False)[0])


class TableEmbeddings:
    """Encoder outputs e for every (source table, dim) pair that can occur:
    the task's tables at their own dim and every dim reachable by halving
    (App. B.1 augmentation PAPER.md:200)."""

    def __init__(self, weights, task):
        self.weights = weights
        self.task = task
        self.e: Dict[Tuple[int, int], np.ndarray] = {}
        for s in range(task.T):
            d = int(task.dims[s])
            while True:
                x = featurize(d, int(task.hash[s]), float(task.pooling[s]), float(task.skew[s]))
                self.e[(s, d)] = encode(weights, x)
                if d % 8 != 0:
                    break
                d //= 2

    def get(self, key: Tuple[int, int]) -> np.ndarray:
        return self.e[key]


def canonical(members: Iterable[Tuple[int, int]]) -> Tuple[Tuple[int, int], ...]:
    """Canonical order of a multiset of (source, dim): ascending (source, dim)."""
    return tuple(sorted(members))


def compute_cost(weights, emb: TableEmbeddings, members: Iterable[Tuple[int, int]]) -> float:
    """O4.  Computation cost of the set of tables on one GPU:
    "element-wise sum of all the table representations" then the head MLP.
    The sum is taken in canonical order so the value is a function of the
    multiset alone.  C(empty) = 0 (reading R4)."""
    key = canonical(members)
    if len(key) == 0:
        return 0.0
    s = np.zeros(32, dtype=np.float64)
    for m in key:
        s = s + emb.get(m)
    return head(weights, s)


def comm_costs(layers, starts: np.ndarray, devdims: np.ndarray,
               start_scale: float, dim_scale: float) -> np.ndarray:
    """O5.  Communication cost MLP "128-64-32-16" mapping the
    per-GPU starting timestamps and data sizes to per-GPU costs:
    input [starts/start_scale, devdims/dim_scale] (2D), output D."""
    x = np.concatenate([np.asarray(starts, np.float64) / start_scale,
                        np.asarray(devdims, np.float64) / dim_scale])
    return mlp(layers, x, relu_last=False)


def reduce_plan(comp: np.ndarray, fwd: np.ndarray, bwd: np.ndarray, sum_of_max: bool = False) -> float:
    """The reduction of O6 over devices.  Reading R11 (default): the maximum
    over devices of the per-device sum comp + fwd + bwd ("the
    maximum cost across devices").  Alternative (``sum_of_max``, flag
    NS_R11_SUM_OF_MAX): "summing up the predicted computation,
    forward communication, and backward communication costs" read as the sum
    of the three per-term maxima."""
    if sum_of_max:
        return float(comp.max() + fwd.max() + bwd.max())
    return float((comp + fwd + bwd).max())


def plan_cost(weights, emb: TableEmbeddings, tables: List[Tuple[int, int]],
              assign: Sequence[int], D: int, abs_starts: bool = False, sum_of_max: bool = False):
    """O6.  Simulated embedding cost f(c, t): "summing up the
    predicted computation, forward communication, and backward communication
    costs", reduced by the maximum over devices (reading R11,
    ``reduce_plan``).  Forward starts are the relative compute delays
    comp - min(comp) (reading R10; ``abs_starts``: the absolute compute costs,
    flag NS_R10_ABS_STARTS), backward starts are zero.

    ``tables`` is the post-split table list [(source, dim)], ``assign[i]`` the
    device of table i.  Returns (cost, comp[D], fwd[D], bwd[D], devdim[D]).
    """
    members: List[List[Tuple[int, int]]] = [[] for _ in range(D)]
    devdim = np.zeros(D, dtype=np.float64)
    for i, d in enumerate(assign):
        members[int(d)].append(tables[i])
        devdim[int(d)] += tables[i][1]
    comp = np.array([compute_cost(weights, emb, members[d]) for d in range(D)])
    starts = comp if abs_starts else comp - comp.min()
    fwd = comm_costs(weights.comm_fwd, starts, devdim, weights.start_scale, weights.dim_scale)
    bwd = comm_costs(weights.comm_bwd, np.zeros(D), devdim, weights.start_scale, weights.dim_scale)
    return reduce_plan(comp, fwd, bwd, sum_of_max), comp, fwd, bwd, devdim
