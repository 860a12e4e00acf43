"""Embedding-bag forward / backward+SGD (single-GPU
half), fp64 -- TEST INFRASTRUCTURE ONLY.

The paper measures a device's computation cost by running the fused
embedding-bag operation of its tables, forward and backward (App. A.2,
PAPER.md:594-600; FBGEMM).  What that operation computes has a plain
definition, written out here:

* forward, sum pooling: out[b][col_t + j] = sum_{i in bag(b, t)} W_t[i][j];
* backward with the optimizer fused (SGD, learning rate lr):
  W_t[i] <- W_t[i] - lr * sum over the occurrences of row i in the bags of
  table t of grad_out[b][col_t ...];
* the two all-to-alls of the model-parallel step (each GPU
  obtains the embeddings of its samples from every GPU's tables "through an
  all-to-all communication"; "the gradients are sent back to the GPUs with
  another all-to-all"), with R ranks, rank q owning samples q*Bl ..
  (q+1)*Bl - 1 (Bl = B / R) and rank r the tables of columns
  [c_r, c_r + cols[r]) of the global pooled matrix: rank q receives, for
  every r, the block pooled[q*Bl:(q+1)*Bl, c_r:c_r+cols[r]] (rank-blocked, r
  ascending); the backward sends block r of each rank's gradient back to
  rank r, which stacks the blocks of ranks q = 0 .. R-1 as its rows.
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


def _col_starts(cols: Sequence[int]) -> List[int]:
    c, out = 0, []
    for n in cols:
        out.append(c)
        c += int(n)
    return out


def exchange_forward(pooled: np.ndarray, cols: Sequence[int]) -> List[np.ndarray]:
    """Forward all-to-all: per rank q, the flat rank-blocked receive buffer
    (block r = pooled[q*Bl:(q+1)*Bl, c_r:c_r+cols[r]], row-major)."""
    R = len(cols)
    B = pooled.shape[0]
    Bl = B // R
    starts = _col_starts(cols)
    out = []
    for q in range(R):
        blocks = [pooled[q * Bl:(q + 1) * Bl, starts[r]:starts[r] + int(cols[r])].reshape(-1) for r in range(R)]
        out.append(np.concatenate(blocks))
    return out


def exchange_backward(grad_recv: Sequence[np.ndarray], cols: Sequence[int]) -> List[np.ndarray]:
    """Backward all-to-all: grad_recv[q] has the forward receive layout of
    rank q; rank r gets [B][cols[r]] with rows q*Bl .. from rank q's block r."""
    R = len(cols)
    Bl = len(grad_recv[0]) // sum(int(c) for c in cols) if sum(cols) else 0
    out = []
    for r in range(R):
        rows = []
        for q in range(R):
            off = Bl * sum(int(c) for c in cols[:r])
            rows.append(np.asarray(grad_recv[q][off:off + Bl * int(cols[r])]).reshape(Bl, int(cols[r])))
        out.append(np.concatenate(rows, axis=0))
    return out
