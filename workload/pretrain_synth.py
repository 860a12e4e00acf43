"""Seeded random draws for pre-training: the table pool,
Alg. 4's combinations and Alg. 5's subsets and uniforms
with App. F's ranges.  Random numbers only -- no method
arithmetic: the placement rule, features, labels and training live in the
oracle (oracle/pretrain.py) and the CUDA path (k_pretrain.cu), which both
consume these arrays.
"""
from __future__ import annotations

import dataclasses

import numpy as np

from .synth import _sample_tables

AUG_DIMS = (4, 8, 16, 32, 64, 128)   # App. F: "we augment the table pool with dimensions {4, ..., 128}"


@dataclasses.dataclass
class Pool:
    dims: np.ndarray     # int32 (the pool's own dims; replaced by the augmentation dims)
    hash: np.ndarray     # int64
    pooling: np.ndarray  # float64
    skew: np.ndarray     # float64

    @property
    def n(self) -> int:
        return int(self.dims.shape[0])


def gen_pool(n: int = 856, seed: int = 91) -> Pool:
    """A synthetic table pool (the paper's DLRM pool has 856 tables
    / PAPER.md Table 5) with the G1 recipe of workload/synth.py."""
    rng = np.random.default_rng(seed)
    dims, hash_, pooling, skew = _sample_tables(rng, n, 128)
    return Pool(dims, hash_, pooling, skew)


def gen_combinations(n_aug: int, n: int, t_min: int = 1, t_max: int = 15, seed: int = 92):
    """Alg. 4 lines 3-6: T ~ U{t_min..t_max}, then T distinct augmented tables
    uniformly.  Returns (off [n+1] int32, idx [off[n]] int32)."""
    rng = np.random.default_rng(seed)
    T = rng.integers(t_min, t_max + 1, size=n)
    off = np.zeros(n + 1, np.int32)
    np.cumsum(T, out=off[1:])
    idx = np.concatenate([rng.choice(n_aug, size=int(t), replace=False) for t in T]).astype(np.int32)
    return off, idx


@dataclasses.dataclass
class PlacementDraws:
    off: np.ndarray      # [n+1] int32
    idx: np.ndarray      # [rows] int32 augmented-table indices (line 5)
    p: np.ndarray        # [n] greedy probability (line 7)
    u: np.ndarray        # [rows] p' of the k-th table in the SORTED order (line 9)
    r: np.ndarray        # [rows] uniform for the random device of the k-th sorted table (line 14)
    starts: np.ndarray   # [n][D] communication start timestamps, ms (App. F: 0-20 ms)


def gen_placement_draws(n_aug: int, n: int, D: int, t_min: int, t_max: int, start_ms: float = 20.0,
                        seed: int = 93) -> PlacementDraws:
    """Alg. 5's random inputs: T ~ U{t_min..t_max} (App. F: 10-60 tables on 4
    GPUs, 20-120 on 8), T distinct augmented tables, p ~ U[0,1], per table
    p' ~ U[0,1] and the random-choice uniform, starts ~ U[0, start_ms]."""
    rng = np.random.default_rng(seed)
    T = rng.integers(t_min, t_max + 1, size=n)
    off = np.zeros(n + 1, np.int32)
    np.cumsum(T, out=off[1:])
    idx = np.concatenate([rng.choice(n_aug, size=int(t), replace=False) for t in T]).astype(np.int32)
    rows = int(off[-1])
    return PlacementDraws(off, idx, rng.uniform(0.0, 1.0, n), rng.uniform(0.0, 1.0, rows),
                          rng.uniform(0.0, 1.0, rows), rng.uniform(0.0, start_ms, (n, D)))


def init_params(widths, seed: int) -> np.ndarray:
    """torch.nn.Linear-style init U(+-1/sqrt(fan_in)) for W and b, flat in
    the layer order (W [out][in] then b)."""
    rng = np.random.default_rng(seed)
    parts = []
    for i, o in widths:
        bound = 1.0 / np.sqrt(i)
        parts.append(rng.uniform(-bound, bound, size=i * o))
        parts.append(rng.uniform(-bound, bound, size=o))
    return np.concatenate(parts)


def gen_bag_indices(rows: int, pooling: float, skew: float, B: int, rng: np.random.Generator):
    """Embedding-bag inputs of one table: bag lengths
    ~ Poisson(pooling factor) (empty bags possible), row ids Zipf-like with
    exponent = the table's skew (0 = uniform) over the table's rows: rank
    k = floor of the inverse CDF of the continuous power law on [1, rows+1),
    mapped to a row by a fixed multiplicative hash so the hot rows are spread
    over the table.  Returns (offsets [B+1] int32, indices int64)."""
    lens = rng.poisson(pooling, size=B)
    off = np.zeros(B + 1, np.int64)
    np.cumsum(lens, out=off[1:])
    n = int(off[-1])
    u = rng.uniform(0.0, 1.0, size=n)
    H = float(rows)
    if abs(skew - 1.0) < 1e-9:
        k = np.floor(np.exp(u * np.log(H + 1.0)))
    else:
        a = 1.0 - skew
        k = np.floor((((H + 1.0) ** a - 1.0) * u + 1.0) ** (1.0 / a))
    k = np.clip(k.astype(np.int64), 1, rows) - 1
    idx = (k * 2654435761) % rows
    return off.astype(np.int32), idx.astype(np.int64)
