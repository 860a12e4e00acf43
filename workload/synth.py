"""Seeded synthetic workload recipes (generator G1 of SURVEY.md §8(d)).

Everything here is random-number generation only.  The shapes and value
distributions follow the paper's task construction and are documented in
DESIGN.md §"Input recipe":

* table dims ~ U{4, 8, ..., max_dim}            (Table 5)
* hash sizes ~ round(logU[1e4, 1e7])             (invented, calibrated; SURVEY.md App. A probe 4)
* pooling ~ logU[1, 60] (mean ~14.4, paper: 15)  (Table 7)
* skew ~ U[0, 2]  ("indices distribution" as a scalar)
* per-device memory cap 4 GiB
* task rejection: sum(bytes) > 0.9 * D * cap; table-wise configs also reject a
  single table larger than the cap (it could never be placed without a split).

Cost-model weights are random-init with the paper's architecture
(App. C: compute "128-32" encoder + "32-64" head, comm
"128-64-32-16"):

* ``mono``   Kaiming-uniform U(+-1/sqrt(fan_in)) for weights and biases, with
             |.| on head H1, H2, hb2 and on each comm model's last layer, so
             predicted costs are >= 0 and monotone in the table set.
* ``signed`` the same without |.|.
* ``inv``    mono, but comm layer 1 has one shared column for the start block
             and one for the dim block and the last comm layer has equal rows:
             per-device comm is identical, so plan cost is exactly invariant
             under device relabelling (test-only).
* ``lin``    the compute model is C(S) = a * sum(dim) + b (the encoder passes
             dim through, the head is linear on it); comm weights are zero.
             Used to pin the greedy against textbook LPT (test-only).
* ``zero``   all weights zero, biases random (test-only: bias-only outputs).

The table-size rule used by the rejection test (bytes = hash * dim * 4, fp32,
no optimiser state) is SURVEY.md reading R7 / SPEC.md:59.
"""
from __future__ import annotations

import dataclasses
from typing import Dict, List, Tuple

import numpy as np

GiB = 1 << 30

# name -> recipe.  Index i of each task uses seed 1000 * cfg_id + i.
CONFIGS: Dict[str, dict] = {
    # BASELINE.json configs[0..4]; SURVEY.md §8(d) table.
    "C1": dict(cfg_id=1, T=10, D=2, cap=4 * GiB, max_dim=128, mode="tablewise",
               N=10, K=3, L=0, M=3, reject_single=True),
    "C2": dict(cfg_id=2, T=40, D=4, cap=4 * GiB, max_dim=128, mode="tablewise",
               N=10, K=3, L=0, M=11, reject_single=True),
    "C3": dict(cfg_id=3, T=80, D=8, cap=4 * GiB, max_dim=128, mode="columnwise",
               N=10, K=10, L=10, M=11, reject_single=False),
    "C4": dict(cfg_id=4, T=200, D=8, cap=8 * GiB, max_dim=128, mode="columnwise",
               N=10, K=3, L=10, M=51, reject_single=False),
    "C5": dict(cfg_id=5, T=1000, D=128, cap=4 * GiB, max_dim=128, mode="columnwise",
               N=10, K=3, L=10, M=11, reject_single=False),
    # SURVEY §8(f) F4 stress shape beyond the paper's production model (nearly a
    # thousand tables on 128 GPUs): 4000 tables on 128 devices,
    # the cap raised to 16 GiB so the same table recipe fits (2 TiB in total,
    # "multi-terabyte memory").  Not a BASELINE.json config.
    "C6": dict(cfg_id=6, T=4000, D=128, cap=16 * GiB, max_dim=128, mode="columnwise",
               N=10, K=3, L=10, M=11, reject_single=False),
}


@dataclasses.dataclass
class Task:
    dims: np.ndarray      # int32 [T]
    hash: np.ndarray      # int64 [T]
    pooling: np.ndarray   # float64 [T]
    skew: np.ndarray      # float64 [T]
    D: int
    cap: int              # bytes per device
    seed: int

    @property
    def T(self) -> int:
        return int(self.dims.shape[0])


@dataclasses.dataclass
class Weights:
    """Layer lists of (W [out, in], b [out]) in float64, torch.nn.Linear layout."""
    enc: List[Tuple[np.ndarray, np.ndarray]]
    head: List[Tuple[np.ndarray, np.ndarray]]
    comm_fwd: List[Tuple[np.ndarray, np.ndarray]]
    comm_bwd: List[Tuple[np.ndarray, np.ndarray]]
    D: int
    start_scale: float = 20.0    # ms; starts sampled in [0, 20] ms
    dim_scale: float = 1024.0
    kind: str = "mono"


def _sample_tables(rng: np.random.Generator, T: int, max_dim: int):
    dims = 4 * rng.integers(1, max_dim // 4 + 1, size=T)
    hash_ = np.rint(np.exp(rng.uniform(np.log(1e4), np.log(1e7), size=T))).astype(np.int64)
    pooling = np.exp(rng.uniform(np.log(1.0), np.log(60.0), size=T))
    skew = rng.uniform(0.0, 2.0, size=T)
    return dims.astype(np.int32), hash_, pooling.astype(np.float64), skew.astype(np.float64)


def gen_task(cfg: str, i: int, T: int | None = None, D: int | None = None) -> Task:
    """Task i of config ``cfg`` (deterministic in (cfg, i))."""
    c = CONFIGS[cfg]
    T = c["T"] if T is None else T
    D = c["D"] if D is None else D
    seed = 1000 * c["cfg_id"] + i
    rng = np.random.default_rng(seed)
    for _ in range(100000):
        dims, hash_, pooling, skew = _sample_tables(rng, T, c["max_dim"])
        sizes = hash_ * dims.astype(np.int64) * 4
        if sizes.sum() > 0.9 * D * c["cap"]:
            continue
        if c["reject_single"] and sizes.max() > c["cap"]:
            continue
        return Task(dims, hash_, pooling, skew, D, int(c["cap"]), seed)
    raise RuntimeError("task rejection loop did not terminate")


def gen_tasks(cfg: str, n: int, start: int = 0, **kw) -> List[Task]:
    return [gen_task(cfg, start + i, **kw) for i in range(n)]


def _linear(rng, fan_in: int, fan_out: int):
    bound = 1.0 / np.sqrt(fan_in)
    W = rng.uniform(-bound, bound, size=(fan_out, fan_in))
    b = rng.uniform(-bound, bound, size=(fan_out,))
    return W, b


def gen_weights(D: int, kind: str = "mono", seed: int = 7, F: int = 5) -> Weights:
    """Cost-model weights: compute model seed ``seed``, comm fwd seed+1, bwd seed+2."""
    rc = np.random.default_rng(seed)
    enc = [_linear(rc, F, 128), _linear(rc, 128, 32)]
    head = [_linear(rc, 32, 64), _linear(rc, 64, 1)]
    comm = []
    for s in (seed + 1, seed + 2):
        rr = np.random.default_rng(s)
        widths = [2 * D, 128, 64, 32, 16, D]
        comm.append([_linear(rr, widths[j], widths[j + 1]) for j in range(5)])
    if kind in ("mono", "inv"):
        head = [(np.abs(head[0][0]), head[0][1]), (np.abs(head[1][0]), np.abs(head[1][1]))]
        comm = [m[:4] + [(np.abs(m[4][0]), np.abs(m[4][1]))] for m in comm]
    if kind == "inv":
        new = []
        for m in comm:
            W1, b1 = m[0]
            W1 = W1.copy()
            W1[:, :D] = W1[:, :1]          # one shared column for the start block
            W1[:, D:] = W1[:, D:D + 1]     # one shared column for the dim block
            W5, b5 = m[4]
            W5 = np.repeat(W5[:1], D, axis=0)
            b5 = np.repeat(b5[:1], D)
            new.append([(W1, b1)] + m[1:4] + [(W5, b5)])
        comm = new
    elif kind == "lin":
        a = 0.01 + abs(float(rc.uniform(0.0, 0.05)))
        b = 0.5 + abs(float(rc.uniform(0.0, 1.0)))
        E1 = np.zeros((128, F)); E1[0, 0] = 128.0          # h0 = relu(dim)
        E2 = np.zeros((32, 128)); E2[0, 0] = 1.0            # e0 = dim
        H1 = np.zeros((64, 32)); H1[0, 0] = 1.0             # hidden0 = sum(dim)
        H2 = np.zeros((1, 64)); H2[0, 0] = a
        enc = [(E1, np.zeros(128)), (E2, np.zeros(32))]
        head = [(H1, np.zeros(64)), (H2, np.array([b]))]
        comm = [[(np.zeros_like(W), np.zeros_like(bb)) for (W, bb) in m] for m in comm]
    elif kind == "zero":
        enc = [(np.zeros_like(W), b) for (W, b) in enc]
        head = [(np.zeros_like(W), b) for (W, b) in head]
        comm = [[(np.zeros_like(W), b) for (W, b) in m] for m in comm]
    elif kind not in ("mono", "signed"):
        raise ValueError(kind)
    return Weights(enc=enc, head=head, comm_fwd=comm[0], comm_bwd=comm[1], D=D, kind=kind)


def gen_plans(T_prime: int, D: int, P: int, seed: int) -> np.ndarray:
    """P uniformly random table->device assignments, int8 [P, T_prime]."""
    rng = np.random.default_rng(seed)
    return rng.integers(0, D, size=(P, T_prime)).astype(np.int8)
