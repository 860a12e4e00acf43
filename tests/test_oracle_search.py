"""Pins for oracle/search.py (O7-O12): worked example, grid arithmetic,
textbook LPT special case, exhaustive optima, brute-force beam, cache
neutrality and hit rate, monotonicity in L, infeasibility.  CPU only."""
import math

import numpy as np
import pytest

from conftest import hand_task, hand_weights, small_task
from oracle import brute, model as om, search as osr
from workload.synth import gen_task, gen_weights


# ---------------------------------------------------------------- worked example
def test_hand_example_greedy_grid_search(golden_hand):
    g = golden_hand
    w, task = hand_weights(g), hand_task(g)
    emb = om.TableEmbeddings(w, task)
    exp = g["expected"]
    tables = osr.apply_col_plan(task, [])
    singles = osr.single_costs(w, emb, tables)
    assert osr.cost_order(singles) == exp["order"]
    assert osr.grid_max_dims(132, 2, 2) == exp["grid"]
    r = osr.greedy_grid_search(w, emb, task, [], g["M"])
    assert r.assign == exp["assign"]
    assert r.grid_index == exp["grid_index"]
    assert r.work == exp["work"]
    assert r.cost == pytest.approx(exp["cost"], rel=1e-12)
    assert math.isinf(r.grid_costs[0])


# ------------------------------------------------------------------ grid (T1, T2)
def test_grid_arithmetic():
    # sum of dims 400, D=4, M=11 -> {100, 105, ..., 150}.
    assert osr.grid_max_dims(400, 4, 11) == [100.0 + 5 * i for i in range(11)]
    # M=1 -> single grid point at M_s.
    assert osr.grid_max_dims(400, 4, 1) == [100.0]


# ------------------------------------------------------------- T3: grid = min of M
def test_ggs_is_best_of_independent_greedies():
    w = gen_weights(4, "mono")
    task = gen_task("C2", 4)
    emb = om.TableEmbeddings(w, task)
    r = osr.greedy_grid_search(w, emb, task, [], 5)
    tables = osr.apply_col_plan(task, [])
    order = osr.cost_order(osr.single_costs(w, emb, tables))
    costs = []
    for md in osr.grid_max_dims(int(task.dims.sum()), 4, 5):
        g = osr.greedy_place(w, emb, task, tables, order, 4, int(math.floor(md)))
        costs.append(om.plan_cost(w, emb, tables, g.assign, 4)[0] if g.assign else math.inf)
    assert r.cost == min(costs)
    assert r.grid_index == costs.index(min(costs))


# ------------------------------------------------- textbook special case: LPT
def _lpt(dims, D):
    """Textbook LPT multiway partition: sort by size descending (stable),
    each job to the least-loaded machine, lowest index on ties."""
    order = sorted(range(len(dims)), key=lambda i: (-dims[i], i))
    load = [0] * D
    a = [-1] * len(dims)
    for i in order:
        d = min(range(D), key=lambda k: (load[k], k))
        a[i] = d
        load[d] += dims[i]
    return a, load


@pytest.mark.parametrize("seed", range(6))
def test_greedy_reduces_to_lpt_with_linear_cost(seed):
    # With C(S) = a*sum(dim) + b the after-insertion greedy (R5) is LPT on dims
    # (App. E "Dim-based" greedy).
    rng = np.random.default_rng(seed)
    D = 2 + seed % 3
    task = small_task(rng, 25, D, hash_hi=1e5)
    w = gen_weights(D, "lin")
    emb = om.TableEmbeddings(w, task)
    tables = osr.apply_col_plan(task, [])
    order = osr.cost_order(osr.single_costs(w, emb, tables))
    assert [int(task.dims[i]) for i in order] == sorted(task.dims.tolist(), reverse=True)
    g = osr.greedy_place(w, emb, task, tables, order, D, 10**9)
    a_ref, load = _lpt(task.dims.tolist(), D)
    assert g.assign == a_ref
    # greedy-balance bound
    assert max(load) - min(load) <= max(task.dims)
    assert g.work == D * task.T


# -------------------------------------------------- T4: exhaustive optimum bound
@pytest.mark.parametrize("seed", range(8))
def test_ggs_cost_at_least_exhaustive_optimum(seed):
    rng = np.random.default_rng(100 + seed)
    D = 2 + seed % 3
    T = 6 if D < 4 else 5
    task = small_task(rng, T, D)
    w = gen_weights(D, "mono" if seed % 2 == 0 else "signed", seed=7 + seed)
    emb = om.TableEmbeddings(w, task)
    tables = osr.apply_col_plan(task, [])
    best, argset, _ = brute.exhaustive_best(w, emb, task, tables, D)
    r = osr.greedy_grid_search(w, emb, task, [], 11)
    assert r.cost >= best
    if r.cost == best:
        assert r.assign in argset


def test_plans_respect_constraints():
    w = gen_weights(8, "mono")
    task = gen_task("C3", 1)
    emb = om.TableEmbeddings(w, task)
    r = osr.beam_search(w, emb, task, N=3, K=2, L=2, M=3)
    assert math.isfinite(r.cost)
    tables = osr.apply_col_plan(task, r.col_plan)
    load = [0] * 8
    dd = [0] * 8
    for i, d in enumerate(r.assign):
        load[d] += osr.table_bytes(task, tables[i])
        dd[d] += tables[i][1]
    assert max(load) <= task.cap
    md = osr.grid_max_dims(int(task.dims.sum()), 8, 3)[r.grid_index]
    assert max(dd) <= math.floor(md)
    # T8: reported cost == cost recomputed from scratch on the returned plan
    assert om.plan_cost(w, emb, tables, r.assign, 8)[0] == r.cost


# ----------------------------------------------------- T5: beam vs brute force
@pytest.mark.parametrize("seed", range(5))
def test_beam_without_pruning_equals_brute_force(seed):
    rng = np.random.default_rng(200 + seed)
    D = 2 + seed % 2
    task = small_task(rng, 4, D, max_dim=32)
    w = gen_weights(D, "mono", seed=11 + seed)
    emb = om.TableEmbeddings(w, task)
    L = 2
    r = osr.beam_search(w, emb, task, N=100, K=10**6, L=L, M=3)
    b_cost, b_plan = brute.brute_column_search(w, emb, task, L, 3)
    assert r.cost == b_cost
    # with pruning the beam can only be worse or equal
    rp = osr.beam_search(w, emb, task, N=1, K=1, L=L, M=3)
    assert rp.cost >= b_cost


def test_global_best_non_increasing_in_L():
    w = gen_weights(4, "mono")
    task = gen_task("C2", 5, T=16)
    emb = om.TableEmbeddings(w, task)
    costs = [osr.beam_search(w, emb, task, N=3, K=2, L=L, M=3).cost for L in range(4)]
    assert all(b <= a for a, b in zip(costs, costs[1:]))


# ------------------------------------------------- T6 / T15: cache neutral, hit rate
def test_cache_is_result_neutral_and_hits():
    w = gen_weights(4, "mono")
    task = gen_task("C2", 6, T=20)
    emb = om.TableEmbeddings(w, task)
    cache = osr.LifelongCache()
    a = osr.beam_search(w, emb, task, N=10, K=3, L=4, M=11, cache=cache)
    b = osr.beam_search(w, emb, task, N=10, K=3, L=4, M=11)
    assert a.cost == b.cost and a.assign == b.assign and a.col_plan == b.col_plan
    assert a.work == b.work
    # PAPER.md:490 reports 95.4% with the full beam; reading R5 reproduces it
    # (SURVEY.md App. A probe 3).  A shorter beam on a smaller task still
    # sits far above the 0% of "w/o caching".
    assert cache.hit_rate > 0.85


# ----------------------------------------------------- T14: forced split
def test_oversized_table_forces_split():
    rng = np.random.default_rng(3)
    task = small_task(rng, 6, 2, cap=4 << 30, hash_hi=1e5)
    task.dims[0] = 128
    task.hash[0] = 10_000_000          # 128 * 1e7 * 4 B = 5.1 GB > 4 GiB
    w = gen_weights(2, "mono")
    emb = om.TableEmbeddings(w, task)
    r0 = osr.beam_search(w, emb, task, N=3, K=2, L=0, M=3)
    assert math.isinf(r0.cost)
    r1 = osr.beam_search(w, emb, task, N=3, K=2, L=2, M=3)
    assert math.isfinite(r1.cost) and 0 in r1.col_plan


def test_candidates_rule():
    # Alg. 1 line 8: top-N costly then top-N largest, deduplicated, then the
    # unsplittable ones dropped (R14).
    w = gen_weights(8, "mono")
    task = gen_task("C3", 2)
    emb = om.TableEmbeddings(w, task)
    tables = osr.apply_col_plan(task, [])
    singles = osr.single_costs(w, emb, tables)
    c = osr.beam_candidates(task, tables, singles, 10)
    by_cost = sorted(range(task.T), key=lambda i: -singles[i])[:10]
    by_size = sorted(range(task.T), key=lambda i: -osr.table_bytes(task, tables[i]))[:10]
    assert set(c) == {i for i in set(by_cost) | set(by_size) if tables[i][1] % 8 == 0}
    assert len(c) == len(set(c))


def test_determinism():
    w = gen_weights(4, "mono")
    task = gen_task("C2", 7, T=14)
    emb = om.TableEmbeddings(w, task)
    a = osr.beam_search(w, emb, task, N=4, K=2, L=2, M=5)
    b = osr.beam_search(w, emb, task, N=4, K=2, L=2, M=5)
    assert (a.cost, a.col_plan, a.assign, a.work) == (b.cost, b.col_plan, b.assign, b.work)


# ------------------------------------------- worked beam example (hand-derived)
def _f(x):
    return math.inf if x == "inf" else float(x)


@pytest.fixture
def golden_beam():
    from conftest import load_golden
    return load_golden("beam_example.json")


def test_beam_example_split_appends_to_end(golden_beam):
    # the second half goes to the END of the table list
    g = golden_beam
    task = hand_task(g)
    for c, lst in g["expected"]["split_lists"].items():
        assert osr.apply_col_plan(task, eval(c)) == [tuple(e) for e in lst], c


def test_beam_example_candidates(golden_beam):
    # Alg. 1 line 8: costly list first, then the largest not yet listed
    g = golden_beam
    w, task = hand_weights(g), hand_task(g)
    emb = om.TableEmbeddings(w, task)
    for c, exp in g["expected"]["candidates"].items():
        tables = osr.apply_col_plan(task, eval(c))
        singles = osr.single_costs(w, emb, tables)
        assert osr.beam_candidates(task, tables, singles, g["N"]) == exp, c
    assert osr.single_costs(w, emb, osr.apply_col_plan(task, [])) == g["expected"]["single_costs"]


def test_beam_example_levels_and_result(golden_beam):
    # Alg. 1 lines 13-20: generation order, top-K by
    # (cost, generation) with +inf children, strict-< global best
    g = golden_beam
    w, task = hand_weights(g), hand_task(g)
    emb = om.TableEmbeddings(w, task)
    e = g["expected"]
    trace = []
    r = osr.beam_search(w, emb, task, N=g["N"], K=g["K"], L=g["L"], M=g["M"], trace=trace)
    assert len(trace) == g["L"]
    for lvl, exp in enumerate(e["level_children"]):
        got = [(c, col) for c, _, col in trace[lvl]["children"]]
        assert got == [(_f(c), col) for c, col in exp], lvl
        assert trace[lvl]["beam"] == e["beams"][lvl], lvl
    assert r.cost == e["cost"]
    assert r.col_plan == e["col_plan"]
    assert r.assign == e["assign"]
    assert r.grid_index == e["grid_index"]
    assert r.work == e["work"]
    assert r.n_plans == e["n_plans"]
    assert r.level_best == [_f(x) for x in e["level_best"]]
    for c, a in e["children_assign"].items():
        assert osr.greedy_grid_search(w, emb, task, eval(c), g["M"]).assign == a, c


def test_no_dim_cap_reading():
    # Table 3 "w/o greedy grid search", reading R8b: no
    # dimension threshold.  With the textbook linear cost it is plain LPT on
    # all tables; with the threshold (M = 1, R8) the tight cap can strand.
    rng = np.random.default_rng(9)
    task = small_task(rng, 18, 3, hash_hi=1e5)
    w = gen_weights(3, "lin")
    emb = om.TableEmbeddings(w, task)
    r = osr.greedy_grid_search(w, emb, task, [], 1, dim_cap=False)
    a_ref, _ = _lpt(task.dims.tolist(), 3)
    assert r.assign == a_ref and r.work == 3 * task.T
    with pytest.raises(ValueError):
        osr.greedy_grid_search(w, emb, task, [], 3, dim_cap=False)
    # never fewer feasible tasks than the tightest threshold (a superset of placements is allowed)
    w = gen_weights(4, "mono")
    n_cap = n_free = 0
    for i in range(12):
        t = gen_task("C2", 40 + i, T=14)
        e = om.TableEmbeddings(w, t)
        n_cap += math.isfinite(osr.greedy_grid_search(w, e, t, [], 1).cost)
        n_free += math.isfinite(osr.greedy_grid_search(w, e, t, [], 1, dim_cap=False).cost)
    assert n_free >= n_cap and n_free == 12


def test_candidates_splittable_only_reading(golden_hand):
    # R14 alternative (flag NS_R14_SPLITTABLE): rank only splittable tables.
    # Hand example tables a (dim 60, unsplittable: 60 % 8 = 4), b (40), t (32),
    # single costs 1.35 / 1.90 / 1.32, bytes proportional to dim (equal hash).
    # N = 1, literal: by cost [b], by size [a] -> [b, a] -> a dropped -> [b];
    # N = 1, splittable only: by cost [b], by size [b] -> [b].
    # N = 2, literal: by cost [b, a], by size [a, b] -> [b, a] -> [b];
    # N = 2, splittable only: by cost [b, t], by size [b, t] -> [b, t].
    g = golden_hand
    w, task = hand_weights(g), hand_task(g)
    emb = om.TableEmbeddings(w, task)
    tables = osr.apply_col_plan(task, [])
    singles = osr.single_costs(w, emb, tables)
    assert osr.beam_candidates(task, tables, singles, 1) == [1]
    assert osr.beam_candidates(task, tables, singles, 1, splittable_only=True) == [1]
    assert osr.beam_candidates(task, tables, singles, 2) == [1]
    assert osr.beam_candidates(task, tables, singles, 2, splittable_only=True) == [1, 2]
