"""Exhaustive enumerators -- TEST INFRASTRUCTURE ONLY (pins).

These loops deliberately do not reuse the greedy or beam code: they enumerate
every placement / column plan and score each one with O6 or
O8, so that the search's results can be checked against an exact optimum on
tiny inputs.
"""
from __future__ import annotations

import itertools
from typing import List, Tuple

from .model import plan_cost
from .search import apply_col_plan, greedy_grid_search, table_bytes


def all_placements(task, tables, D: int, respect_memory: bool = True):
    """Yield every assignment in D^T' (lexicographic), optionally only those
    whose per-device bytes fit the cap."""
    n = len(tables)
    sizes = [table_bytes(task, t) for t in tables]
    for a in itertools.product(range(D), repeat=n):
        if respect_memory:
            load = [0] * D
            for i, d in enumerate(a):
                load[d] += sizes[i]
            if max(load) > task.cap:
                continue
        yield list(a)


def exhaustive_best(weights, emb, task, tables, D: int, respect_memory: bool = True):
    """Exact argmin of f over all (memory-feasible) placements: (cost, argmin
    set as list of assignments, all costs)."""
    best = float("inf")
    arg: List[List[int]] = []
    costs = []
    for a in all_placements(task, tables, D, respect_memory):
        c = plan_cost(weights, emb, tables, a, D)[0]
        costs.append(c)
        if c < best:
            best, arg = c, [a]
        elif c == best:
            arg.append(a)
    return best, arg, costs


def all_column_plans(task, L: int) -> List[List[int]]:
    """Every ordered sequence of legal splits of length 0..L (each step must
    split a table whose current dim % 8 == 0)."""
    out: List[List[int]] = [[]]
    frontier: List[List[int]] = [[]]
    for _ in range(L):
        nxt = []
        for c in frontier:
            tables = apply_col_plan(task, c)
            for i, (_, d) in enumerate(tables):
                if d % 8 == 0:
                    nxt.append(c + [i])
        out.extend(nxt)
        frontier = nxt
    return out


def brute_column_search(weights, emb, task, L: int, M: int, hi: float = 1.5) -> Tuple[float, List[int]]:
    """min over every column plan of length <= L of GreedyGridSearch(c)."""
    best, arg = float("inf"), None
    for c in all_column_plans(task, L):
        r = greedy_grid_search(weights, emb, task, c, M, hi)
        if r.cost < best:
            best, arg = r.cost, c
    return best, arg
