"""Embedding-bag forward / backward+SGD (single-GPU
half), fp64 -- TEST INFRASTRUCTURE ONLY.

The paper measures a device's computation cost by running the fused
embedding-bag operation of its tables, forward and backward (App. A.2,
PAPER.md:594-600; FBGEMM).  What that operation computes has a plain
definition, written out here:

* forward, sum pooling: out[b][col_t + j] = sum_{i in bag(b, t)} W_t[i][j];
* backward with the optimizer fused (SGD, learning rate lr):
  W_t[i] <- W_t[i] - lr * sum over the occurrences of row i in the bags of
  table t of grad_out[b][col_t ...].
"""
from __future__ import annotations

from typing import List, Sequence

import numpy as np


def bag_forward(W: Sequence[np.ndarray], idx: Sequence[np.ndarray], off: Sequence[np.ndarray], B: int) -> np.ndarray:
    cols = [w.shape[1] for w in W]
    out = np.zeros((B, sum(cols)), np.float64)
    c = 0
    for t in range(len(W)):
        Wt = W[t].astype(np.float64)
        for b in range(B):
            rows = idx[t][off[t][b]:off[t][b + 1]]
            if len(rows):
                out[b, c:c + cols[t]] = Wt[rows].sum(axis=0)
        c += cols[t]
    return out


def bag_backward_sgd(W: Sequence[np.ndarray], idx: Sequence[np.ndarray], off: Sequence[np.ndarray],
                     gout: np.ndarray, lr: float) -> List[np.ndarray]:
    out, c = [], 0
    for t in range(len(W)):
        dim = W[t].shape[1]
        Wn = W[t].astype(np.float64).copy()
        for b in range(gout.shape[0]):
            for i in idx[t][off[t][b]:off[t][b + 1]]:
                Wn[i] -= lr * gout[b, c:c + dim].astype(np.float64)
        out.append(Wn)
        c += dim
    return out
