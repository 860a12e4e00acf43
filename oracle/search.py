"""Online search (§3.3), fp64 -- TEST INFRASTRUCTURE ONLY.

O7 column split, O8 GreedyGridSearch (Alg. 2),
O9 BeamSearch (Alg. 1), O10 the literal life-long cache
(PAPER.md:291), O11 decision log, O12 work count.  Ambiguities follow the
readings listed in DESIGN.md §"Readings" (R5-R17); every reading is marked
where it is used.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Dict, List, Optional, Tuple

import numpy as np

from .model import TableEmbeddings, canonical, compute_cost, plan_cost

INF = float("inf")


# --------------------------------------------------------------------------- O7
def apply_col_plan(task, c: List[int]) -> List[Tuple[int, int]]:
    """O7.  PAPER.md:237: "c_i means, in step i, we shard the table of index
    c_i into two halves column-wisely and append the resultant new table to
    the end of the table list".  Entries are (source table, dim); the first
    half stays at index c_i, the second is appended.  A table is splittable
    iff dim % 8 == 0 so both halves keep dim % 4 == 0."""
    tables = [(s, int(task.dims[s])) for s in range(task.T)]
    for ci in c:
        s, d = tables[ci]
        if d % 8 != 0:
            raise ValueError(f"table {ci} with dim {d} is not splittable")
        tables[ci] = (s, d // 2)
        tables.append((s, d // 2))
    return tables


def table_bytes(task, entry: Tuple[int, int]) -> int:
    """Reading R7: fp32 rows, no optimiser state: bytes = hash * dim * 4."""
    s, d = entry
    return int(task.hash[s]) * int(d) * 4


# -------------------------------------------------------------------------- O10
class LifelongCache:
    """O10.  "a life-long hash map as a cache": key = the set of
    tables on a GPU (Alg. 2 line "if the tables in GPU are in global_cache",
    PAPER.md:310), canonical multiset of (source, dim).  Result-neutral."""

    def __init__(self):
        self.table: Dict[tuple, float] = {}
        self.hits = 0
        self.misses = 0

    def cost(self, weights, emb, members) -> float:
        key = canonical(members)
        if key in self.table:
            self.hits += 1
            return self.table[key]
        self.misses += 1
        v = compute_cost(weights, emb, key)
        self.table[key] = v
        return v

    @property
    def hit_rate(self) -> float:
        n = self.hits + self.misses
        return self.hits / n if n else 0.0


# -------------------------------------------------------------------------- O11
@dataclasses.dataclass
class DecisionLog:
    """O11.  Relative top-2 margins of every comparison that picks a winner."""
    margins: List[Tuple[str, float]] = dataclasses.field(default_factory=list)
    exact_ties: int = 0

    def record(self, kind: str, best: float, second: float):
        if not (math.isfinite(best) and math.isfinite(second)):
            return
        if second == best:
            self.exact_ties += 1
            return
        denom = abs(best) if best != 0.0 else 1.0
        self.margins.append((kind, abs(second - best) / denom))

    def min_margin(self, kinds=None) -> float:
        vals = [m for k, m in self.margins if kinds is None or k in kinds]
        return min(vals) if vals else INF


def _cost(weights, emb, members, cache: Optional[LifelongCache]) -> float:
    if cache is not None:
        return cache.cost(weights, emb, members)
    return compute_cost(weights, emb, members)


# --------------------------------------------------------------------------- O8
def grid_max_dims(sum_dim: int, D: int, M: int, hi: float = 1.5) -> List[float]:
    """"we try all the values in [M_s, M_e] with a step size of
    (M_e - M_s)/(M-1) ... M_s [is] the average dimension across device and M_e
    [is] 1.5 * M_s".  M = 1 gives the single point M_s (reading R8).  The
    operation order (one division, one multiply, one subtraction/division,
    one multiply-add written as two roundings) is part of the reading."""
    Ms = float(sum_dim) / float(D)
    Me = hi * Ms
    if M == 1:
        return [Ms]
    step = (Me - Ms) / float(M - 1)
    return [Ms + float(m) * step for m in range(M)]


def single_costs(weights, emb, tables, cache=None) -> List[float]:
    """Alg. 2 line 3 sort key: the cost "predicted by the computation cost
    model" of each table alone, C({t})."""
    return [_cost(weights, emb, [t], cache) for t in tables]


def cost_order(singles: List[float]) -> List[int]:
    """Descending predicted cost, ties by list index (reading R13)."""
    return sorted(range(len(singles)), key=lambda i: (-singles[i], i))


@dataclasses.dataclass
class GreedyResult:
    assign: Optional[List[int]]   # device per list index, None if stranded
    work: int                     # O12: number of candidate scores evaluated


def greedy_place(weights, emb, task, tables, order, D: int, max_dim_floor: int,
                 cache=None, log: Optional[DecisionLog] = None) -> GreedyResult:
    """Alg. 2 lines 6-20 for one max_dim, PAPER.md:289
    step 3: "assign tables one by one to the device with the lowest device
    cost so far subject to the memory and max_dim constraints".

    * candidate GPUs (line 308): bytes_d + bytes_t <= cap and
      dim_d + dim_t <= floor(max_dim) (readings R6, R7);
    * device cost = C(S_d + {t}), the cost after insertion (reading R5);
    * argmin, lowest device index on ties (reading R13);
    * no candidate -> the grid point is infeasible (reading R9).
    """
    members: List[List[Tuple[int, int]]] = [[] for _ in range(D)]
    dimsum = [0] * D
    bsum = [0] * D
    assign = [-1] * len(tables)
    work = 0
    for i in order:
        t = tables[i]
        bt = table_bytes(task, t)
        feas = [d for d in range(D)
                if bsum[d] + bt <= task.cap and dimsum[d] + t[1] <= max_dim_floor]
        work += len(feas)
        if not feas:
            return GreedyResult(None, work)
        scored = sorted((_cost(weights, emb, members[d] + [t], cache), d) for d in feas)
        if log is not None and len(scored) > 1:
            log.record("greedy", scored[0][0], scored[1][0])
        d_star = scored[0][1]
        assign[i] = d_star
        members[d_star].append(t)
        dimsum[d_star] += t[1]
        bsum[d_star] += bt
    return GreedyResult(assign, work)


@dataclasses.dataclass
class GGSResult:
    cost: float
    assign: Optional[List[int]]
    grid_index: int
    work: int
    tables: List[Tuple[int, int]]
    grid_costs: List[float]


def greedy_grid_search(weights, emb, task, c: List[int], M: int, hi: float = 1.5,
                       cache=None, log: Optional[DecisionLog] = None, dim_cap: bool = True,
                       abs_starts: bool = False, sum_of_max: bool = False) -> GGSResult:
    """O8 = Alg. 2 GreedyGridSearch.

    Line 2: build the T' = T + |c| column-sharded tables; line 3: sort them in
    descending predicted cost; lines 4-21: for each of the M max_dim values
    run the greedy placement and evaluate the completed plan with the cost
    models (PAPER.md:289 step 4).  Lines 316-318 are mis-nested in the paper;
    read as "best completed plan over the grid points, lowest grid index on
    ties" (reading R12).

    ``dim_cap=False`` is Table 3's "w/o greedy grid search" ("not
    grid-searching the table dimension threshold"; reading
    R8b): one greedy placement with no dimension threshold (M must be 1).
    """
    if not dim_cap and M != 1:
        raise ValueError("dim_cap=False needs M == 1")
    tables = apply_col_plan(task, c)
    singles = single_costs(weights, emb, tables, cache)
    order = cost_order(singles)
    if log is not None:
        for a, b in zip(order, order[1:]):
            log.record("sort", singles[b], singles[a])
    sum_dim = sum(d for _, d in tables)
    best = GGSResult(INF, None, -1, 0, tables, [])
    finite = []
    for m, md in enumerate(grid_max_dims(sum_dim, task.D, M, hi)):
        cap = int(math.floor(md)) if dim_cap else 10 ** 18
        g = greedy_place(weights, emb, task, tables, order, task.D, cap, cache, log)
        best.work += g.work
        if g.assign is None:
            cost = INF
        else:
            if cache is not None:   # the final per-device evaluations also query C(.)
                for d in range(task.D):
                    mem = [tables[i] for i in range(len(tables)) if g.assign[i] == d]
                    if mem:
                        cache.cost(weights, emb, mem)
            cost = plan_cost(weights, emb, tables, g.assign, task.D, abs_starts, sum_of_max)[0]
            finite.append((cost, tuple(g.assign)))
        best.grid_costs.append(cost)
        if cost < best.cost:
            best.cost, best.assign, best.grid_index = cost, g.assign, m
    if log is not None and best.assign is not None:
        others = [c_ for c_, a in finite if a != tuple(best.assign)]
        if others:
            log.record("grid", best.cost, min(others))
    return best


# --------------------------------------------------------------------------- O9
def beam_candidates(task, tables, singles, N: int, splittable_only: bool = False) -> List[int]:
    """Alg. 1 line 8: "merging the top N costly tables and the
    top N tables with the largest sizes with duplicates removed".  Costly =
    single-table predicted cost, order (-cost, index); largest = (-bytes,
    index); then tables that cannot be halved (dim % 8 != 0) are dropped
    (reading R14).  ``splittable_only`` (flag NS_R14_SPLITTABLE): rank only
    the splittable tables, so up to N of each kind survive."""
    n = len(tables)
    pool = [i for i in range(n) if tables[i][1] % 8 == 0] if splittable_only else list(range(n))
    by_cost = sorted(pool, key=lambda i: (-singles[i], i))[:N]
    by_size = sorted(pool, key=lambda i: (-table_bytes(task, tables[i]), i))[:N]
    cand = list(by_cost) + [i for i in by_size if i not in by_cost]
    return [i for i in cand if tables[i][1] % 8 == 0]


@dataclasses.dataclass
class BeamResult:
    cost: float
    col_plan: List[int]
    assign: Optional[List[int]]
    grid_index: int
    work: int
    n_plans: int                 # column plans evaluated (incl. [])
    level_best: List[float]      # best cost among each level's children


def beam_search(weights, emb, task, N: int, K: int, L: int, M: int, hi: float = 1.5,
                cache=None, log: Optional[DecisionLog] = None,
                trace: Optional[list] = None, dim_cap: bool = True, abs_starts: bool = False,
                sum_of_max: bool = False, splittable_only: bool = False) -> BeamResult:
    """O9 = Alg. 1 BeamSearch.

    The empty column plan is evaluated first and is the initial global best
    (reading R15; L = 0 is "w/o beam search").  For each level, every beam plan
    (in beam order) is extended by each of its candidate tables (Alg. 1 lines
    9-12); each extension is scored by GreedyGridSearch; the global best is
    replaced on a strictly lower cost (lines 13-16, earliest wins).  The next
    beam is the K lowest (cost, generation index) plans of the level (line 20;
    generation index = (beam rank, candidate rank), reading R13), infeasible
    plans having cost +inf (reading R16); duplicates are kept (reading R17).
    ``trace`` (optional list) receives one record per level: the candidates
    of every beam plan, the children as (cost, generation index, column
    plan) in evaluation order, and the next beam -- introspection only.
    """
    r0 = greedy_grid_search(weights, emb, task, [], M, hi, cache, log, dim_cap, abs_starts, sum_of_max)
    best = BeamResult(r0.cost, [], r0.assign, r0.grid_index, r0.work, 1, [])
    beam: List[List[int]] = [[]]
    for _level in range(L):
        children = []
        cands = []
        for b, cp in enumerate(beam):
            tables = apply_col_plan(task, cp)
            singles = single_costs(weights, emb, tables, cache)
            cands.append(beam_candidates(task, tables, singles, N, splittable_only))
            for j, t in enumerate(cands[-1]):
                col = cp + [t]
                r = greedy_grid_search(weights, emb, task, col, M, hi, cache, log, dim_cap, abs_starts, sum_of_max)
                best.work += r.work
                best.n_plans += 1
                children.append((r.cost, (b, j), col))
                if r.cost < best.cost:
                    if log is not None:
                        log.record("global", r.cost, best.cost)
                    best.cost, best.col_plan = r.cost, col
                    best.assign, best.grid_index = r.assign, r.grid_index
        evaluated = list(children)
        children.sort(key=lambda x: (x[0], x[1]))
        if log is not None and len(children) > K:
            log.record("topk", children[K - 1][0], children[K][0])
        best.level_best.append(children[0][0] if children else INF)
        beam = [col for _, _, col in children[:K]]
        if trace is not None:
            trace.append({"candidates": cands, "children": evaluated, "beam": [list(c) for c in beam],
                          "global_best": (best.cost, list(best.col_plan))})
        if not beam:
            break
    return best
