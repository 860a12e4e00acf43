"""GPU oracle identity on the full-size search paths (VERDICT r1 "next
round" 1(b)): the decisions of the CUDA path against the fp64 oracle's on the
long-list order / candidate kernels (T' > 256), the wide greedy (D = 128),
full-depth beams (C3 K = 10 L = 10, C4 L = 10 M = 51) and ragged batches that
mix one long task into short ones (the list-length switch is batch-wide).

Expected values for the minutes-long cases come from
tests/golden/oracle_full.json, written by tools/make_oracle_fixtures.py (which
calls only oracle/); the short cases run the oracle here.  Tolerance: fp64 on
both sides -> costs within 1e-12 relative and identical integers, unless the
oracle's decision log has a margin below 1e-12, in which case the returned
plan is certified instead (tests/certify.py)."""
import math

import numpy as np
import pytest

from certify import certify_plan
from conftest import load_golden, small_task
from oracle import model as om, search as osr
from workload.synth import CONFIGS, gen_task, gen_tasks, gen_weights

pytestmark = pytest.mark.gpu

RTOL = 1e-12
FIX = load_golden("oracle_full.json")["cases"]


@pytest.fixture(scope="module")
def ns():
    import torch
    assert torch.cuda.is_available()
    import paper_2305_01868_b200 as ns
    return ns


@pytest.fixture(scope="module")
def ctx(ns):
    c = ns.ns_create(0)
    yield c
    ns.ns_destroy(c)


def _f(x):
    return math.inf if x == "inf" else float(x)


def _run(ns, ctx, tasks, w, mode, N, K, L, M, greedy=0, dim_cap=True):
    ns.ns_load_cost_models(ctx, w)
    desc, off, caps = ns.table_descs(tasks)
    tabs = ns.ns_featurize_tables(ctx, desc, off, caps)
    try:
        if mode == "tablewise":
            return ns.ns_shard_tablewise(ctx, tabs, w.D, M=M, greedy=greedy, no_dim_cap=not dim_cap)
        return ns.ns_shard_columnwise(ctx, tabs, w.D, N=N, K=K, L=L, M=M, greedy=greedy, no_dim_cap=not dim_cap)
    finally:
        tabs.free()


def _compare(out, i, task, w, exp, min_margin, M, dim_cap=True):
    """Exact identity when the oracle is tie-free at fp64 resolution, else
    certify the returned plan."""
    nc = int(out["n_col"][i]) if out.get("n_col") is not None else 0
    col = out["col_plan"][i, :nc].tolist() if nc else []
    cost = float(out["cost"][i])
    if min_margin >= RTOL:
        assert col == exp["col_plan"], "column plan"
        ec = _f(exp["cost"])
        assert (math.isinf(cost) and math.isinf(ec)) or abs(cost - ec) <= RTOL * abs(ec), (cost, ec)
        assert int(out["n_scores"][i]) == exp["work"], "work W"
        if exp["assign"] is not None:
            assert int(out["grid_index"][i]) == exp["grid_index"]
            assert out["assign"][i, :task.T + nc].tolist() == exp["assign"], "assignment"
        return "identical"
    if math.isinf(cost):
        assert math.isinf(_f(exp["cost"]))
        return "infeasible"
    certify_plan(w, task, col, out["assign"][i, :task.T + nc].tolist(), int(out["grid_index"][i]), cost, M,
                 dim_cap=dim_cap)
    return "certified"


@pytest.mark.parametrize("greedy", [0, 1])
@pytest.mark.parametrize("name", sorted(FIX))
def test_fullsize_against_oracle_fixture(ns, ctx, name, greedy):
    """greedy 0 = auto (a single task: the latency kernels), 1 = the grouped
    kernels (k_greedy_dedup for D <= 16, k_greedy_wgrp88 for D = 128)."""
    c = FIX[name]
    task = gen_task(c["config"], c["task_index"], T=c["T"] if c["T"] != CONFIGS[c["config"]]["T"] else None)
    assert task.T == c["T"]
    w = gen_weights(c["D"], "mono")
    out = _run(ns, ctx, [task], w, c["mode"], c["N"], c["K"], c["L"], c["M"], greedy=greedy)
    how = _compare(out, 0, task, w, c["expected"], _f(c["min_margin"]), c["M"])
    assert how == "identical" or _f(c["min_margin"]) < RTOL


def test_fullsize_batched_same_as_single(ns, ctx):
    """The C3 fixtures again as one batch of 2 (grouped greedy, batch-wide
    kernels): identical to the oracle as well."""
    names = ["C3_full_0", "C3_full_1"]
    tasks = [gen_task("C3", FIX[n]["task_index"]) for n in names]
    w = gen_weights(8, "mono")
    out = _run(ns, ctx, tasks, w, "columnwise", 10, 10, 10, 11, greedy=1)
    for i, n in enumerate(names):
        _compare(out, i, tasks[i], w, FIX[n]["expected"], _f(FIX[n]["min_margin"]), 11)


def _oracle_check_batch(out, tasks, w, mode, N, K, L, M, dim_cap=True):
    kinds = {"identical": 0, "certified": 0, "infeasible": 0}
    for i, task in enumerate(tasks):
        emb = om.TableEmbeddings(w, task)
        log = osr.DecisionLog()
        if mode == "tablewise":
            r = osr.greedy_grid_search(w, emb, task, [], M, log=log, dim_cap=dim_cap)
            exp = dict(cost=r.cost, col_plan=[], assign=r.assign, grid_index=r.grid_index, work=r.work)
        else:
            r = osr.beam_search(w, emb, task, N=N, K=K, L=L, M=M, log=log, dim_cap=dim_cap)
            exp = dict(cost=r.cost, col_plan=r.col_plan, assign=r.assign, grid_index=r.grid_index, work=r.work)
        kinds[_compare(out, i, task, w, exp, log.min_margin(), M, dim_cap)] += 1
        # the certificate holds for every returned plan, tie or not
        nc = int(out["n_col"][i]) if out.get("n_col") is not None else 0
        if math.isfinite(out["cost"][i]):
            certify_plan(w, task, out["col_plan"][i, :nc].tolist() if nc else [],
                         out["assign"][i, :task.T + nc].tolist(), int(out["grid_index"][i]),
                         float(out["cost"][i]), M, emb=emb, dim_cap=dim_cap)
    return kinds


@pytest.mark.parametrize("greedy", [1, 2])
def test_ragged_batch_long_task_moves_short_tasks_to_long_list_path(ns, ctx, greedy):
    """One T = 300 task among short ones: the batch's max list length selects
    the CTA-per-plan order and block-argmax candidate kernels for EVERY task,
    so the short tasks (oracle-checkable in seconds) exercise the long-list
    path too."""
    w = gen_weights(4, "mono")
    long_task = small_task(np.random.default_rng(900), 300, 4, hash_hi=1e5)   # T = 300 fits D = 4 at 4 GiB
    tasks = [long_task] + gen_tasks("C2", 11, T=16)
    out = _run(ns, ctx, tasks, w, "tablewise", 0, 0, 0, 11, greedy=greedy)
    k = _oracle_check_batch(out, tasks, w, "tablewise", 0, 0, 0, 11)
    assert k["identical"] >= 10
    out = _run(ns, ctx, tasks, w, "columnwise", 4, 2, 2, 5, greedy=greedy)
    k = _oracle_check_batch(out, tasks, w, "columnwise", 4, 2, 2, 5)
    assert k["identical"] >= 10


def test_near_tie_tasks_are_certified(ns, ctx):
    """Tasks whose oracle log has a margin below 1e-12 are not skipped: the
    returned plan is recomputed (T8), validated and certificate-replayed
    (every returned plan is certified as well).  The 'lin' compute model
    (zero comm) makes exact ties abundant: empty devices and equal dim sums."""
    w = gen_weights(4, "lin")
    tasks = gen_tasks("C2", 12, T=24)
    out = _run(ns, ctx, tasks, w, "tablewise", 0, 0, 0, 11)
    k = _oracle_check_batch(out, tasks, w, "tablewise", 0, 0, 0, 11)
    assert sum(k.values()) == len(tasks)
    out = _run(ns, ctx, tasks, w, "columnwise", 4, 2, 2, 5)
    k = _oracle_check_batch(out, tasks, w, "columnwise", 4, 2, 2, 5)
    assert sum(k.values()) == len(tasks)


@pytest.mark.parametrize("D", [40, 128])
def test_wide_grouped_kernel_bit_identical_to_per_trajectory(ns, ctx, D):
    """k_greedy_wgrp88 (identical trajectories share scores, forks on
    divergence) against k_greedy_wide88 (every trajectory alone): same lane
    layout and summation order, so every output is bit-identical -- costs,
    assignments, grid indices, W -- on C5-shaped batches, table- and
    column-wise, and the executed-score counter is below W.  At D = 128 the
    grouped run takes phase 2 (k_greedy_p2 + k_greedy_replay: closed linear
    form scores, replayed representatives) -- the counters prove it ran."""
    w = gen_weights(D, "mono")
    tasks = gen_tasks("C5", 6, start=20, T=400 if D == 128 else 150, D=D)
    for mode, kw in (("tablewise", {}), ("columnwise", dict(N=4, K=2, L=3))):
        outs = {}
        comp, st = {}, {}
        for g in (1, 2):
            ns.ns_profile(ctx, True)
            outs[g] = _run(ns, ctx, tasks, w, mode, kw.get("N", 0), kw.get("K", 0), kw.get("L", 0), 11, greedy=g)
            st[g] = ns.ns_last_stats(ctx)
            comp[g] = st[g]["scores_computed"]
            ns.ns_profile(ctx, False)
        if D == 128:
            assert st[1]["replay_reps"] > 0 and st[1]["replay_rows"] > 0, (mode, st[1])
            assert 0 < st[1]["scores_linear"] < comp[1], (mode, st[1])
        assert st[2]["replay_reps"] == 0
        for k in ("cost", "assign", "grid_index", "n_scores") + (("n_col", "col_plan") if mode == "columnwise" else ()):
            assert np.array_equal(outs[1][k], outs[2][k]), (mode, k)
        W = int(np.sum(outs[1]["n_scores"]))
        assert comp[2] == W                    # per-trajectory kernel: executed == algorithmic
        assert 0 < comp[1] < W                 # grouped: identical trajectories share scores


# every ablation / sweep variant of tools/ablation.py on
# oracle-checkable tasks (T = 16, D = 4, tables that may exceed the cap):
# identical to the oracle's Alg. 1 / Alg. 2 (or certified at near-ties).
ABLATIONS = [
    ("full", "columnwise", dict(N=4, K=2, L=3, M=5), True),
    ("w/o beam search (L = 0)", "columnwise", dict(N=4, K=2, L=0, M=5), True),
    ("w/o greedy grid search (no dim threshold, R8b)", "columnwise", dict(N=4, K=2, L=3, M=1), False),
    ("w/o greedy grid search, table-wise", "tablewise", dict(N=0, K=0, L=0, M=1), False),
    ("single tightest threshold (M = 1, R8)", "columnwise", dict(N=4, K=2, L=3, M=1), True),
    ("sweep N = 1", "columnwise", dict(N=1, K=2, L=3, M=5), True),
    ("sweep K = 1", "columnwise", dict(N=4, K=1, L=3, M=5), True),
    ("sweep K = 3", "columnwise", dict(N=4, K=3, L=3, M=5), True),
    ("sweep L = 1", "columnwise", dict(N=4, K=2, L=1, M=5), True),
    ("sweep M = 9", "columnwise", dict(N=4, K=2, L=2, M=9), True),
]


@pytest.mark.parametrize("name,mode,hp,dim_cap", ABLATIONS, ids=[a[0] for a in ABLATIONS])
def test_ablation_variants_match_oracle(ns, ctx, name, mode, hp, dim_cap):
    w = gen_weights(4, "mono")
    tasks = [gen_task("C3", 500 + i, T=16, D=4) for i in range(10)]
    out = _run(ns, ctx, tasks, w, mode, hp["N"], hp["K"], hp["L"], hp["M"], dim_cap=dim_cap)
    k = _oracle_check_batch(out, tasks, w, mode, hp["N"], hp["K"], hp["L"], hp["M"], dim_cap=dim_cap)
    assert k["identical"] + k["infeasible"] >= 8, k


@pytest.mark.parametrize("D,M", [(17, 64), (33, 1), (128, 2)])
def test_wide_grouped_edges_against_oracle(ns, ctx, D, M):
    """Edges of the large-D kernels: D = 17 (the first D on the wide path)
    with M = 64 (the grouped kernel's member limit), M = 1 (single-member
    groups), M = 2; grouped and per-trajectory kernels bit-identical and
    equal to the oracle's beam search."""
    w = gen_weights(D, "mono", seed=D)
    rng = np.random.default_rng(D)
    tasks = [small_task(rng, 3 * D, D, hash_hi=2e5) for _ in range(2)]
    outs = [_run(ns, ctx, tasks, w, "columnwise", 3, 2, 2, M, greedy=g) for g in (1, 2)]
    for k in ("cost", "assign", "grid_index", "n_scores", "n_col", "col_plan"):
        assert np.array_equal(outs[0][k], outs[1][k]), k
    kinds = _oracle_check_batch(outs[0], tasks, w, "columnwise", 3, 2, 2, M)
    assert kinds["identical"] + kinds["infeasible"] >= 1, kinds


@pytest.mark.parametrize("T", [256, 257])
def test_order_kernel_switch_boundary(ns, ctx, T):
    """T' = 256 is the last list length on the warp-per-plan order kernel,
    257 the first on the CTA bitonic sort (k_build_order): both equal the
    oracle's GreedyGridSearch (order, assignment, W)."""
    w = gen_weights(16, "mono", seed=3)
    task = small_task(np.random.default_rng(T), T, 16, hash_hi=1e5)
    out = _run(ns, ctx, [task], w, "tablewise", 0, 0, 0, 5)
    kinds = _oracle_check_batch(out, [task], w, "tablewise", 0, 0, 0, 5)
    assert kinds["identical"] + kinds["certified"] == 1


def test_bench_launch_C5_batch(ns, ctx):
    """The bench's headline launch (128 C5 tasks per call: the grouped large-D
    greedy with forks on the work queue) against single-task calls of the
    same tasks (the per-trajectory latency kernels): bit-identical plans,
    costs, grid indices and W for a sample of tasks; two of them certified
    by the oracle (T8, validity, certificate replay)."""
    import bench
    c = CONFIGS["C5"]
    w = gen_weights(128, "mono")
    n = 128
    tasks = gen_tasks("C5", n)
    ns.ns_profile(ctx, True)
    out = _run(ns, ctx, tasks, w, "columnwise", c["N"], c["K"], c["L"], c["M"])
    st = ns.ns_last_stats(ctx)
    ns.ns_profile(ctx, False)
    assert st["replay_reps"] > 0 and st["scores_linear"] > 0, st   # phase 2 ran
    assert bench.CFG == "C5"
    certified = 0
    for i in (0, 3, 37, 101):
        one = _run(ns, ctx, [tasks[i]], w, "columnwise", c["N"], c["K"], c["L"], c["M"])
        for k in ("cost", "n_col", "grid_index", "n_scores"):
            assert one[k][0] == out[k][i], (i, k)
        nc = int(out["n_col"][i])
        assert np.array_equal(one["col_plan"][0, :nc], out["col_plan"][i, :nc])
        assert np.array_equal(one["assign"][0, :1000 + nc], out["assign"][i, :1000 + nc])
        if math.isfinite(out["cost"][i]) and certified < 2:
            certify_plan(w, tasks[i], out["col_plan"][i, :nc].tolist(), out["assign"][i, :1000 + nc].tolist(),
                         int(out["grid_index"][i]), float(out["cost"][i]), c["M"])
            certified += 1
    assert certified == 2


def test_merge_orders_identical_to_rank_sort(ns, ctx, monkeypatch):
    """Beam levels with long lists derive each child's cost order from its
    parent's (k_merge_order: remove the split entry, merge the two halves);
    the result must be the rank sort's (k_build_order, forced with
    NS_SORT_ORDERS) bit for bit -- checked through every output of a
    column-wise C5 batch (ragged: one task cut to 700 tables), plus a table
    list with duplicated tables (equal single costs: ties broken by index)."""
    c = CONFIGS["C5"]
    w = gen_weights(128, "mono")
    tasks = gen_tasks("C5", 12)
    t0 = tasks[5]
    tasks[5] = type(t0)(t0.dims[:700], t0.hash[:700], t0.pooling[:700], t0.skew[:700], t0.D, t0.cap, t0.seed)
    t1 = tasks[7]
    rep = np.concatenate([np.arange(400), np.arange(400)])   # every table twice
    tasks[7] = type(t1)(t1.dims[rep], t1.hash[rep], t1.pooling[rep], t1.skew[rep], t1.D, t1.cap, t1.seed)
    merged = _run(ns, ctx, tasks, w, "columnwise", c["N"], c["K"], c["L"], c["M"])
    monkeypatch.setenv("NS_SORT_ORDERS", "1")
    sorted_ = _run(ns, ctx, tasks, w, "columnwise", c["N"], c["K"], c["L"], c["M"])
    monkeypatch.delenv("NS_SORT_ORDERS")
    for k in ("cost", "n_col", "col_plan", "assign", "grid_index", "n_scores"):
        np.testing.assert_array_equal(np.asarray(merged[k]), np.asarray(sorted_[k]), err_msg=k)
    assert int(np.max(merged["n_col"])) >= 2   # beams deeper than level 1 were taken


READINGS = [("R10 absolute starts", 16, dict(abs_starts=True)),
            ("R11 sum of maxima", 32, dict(sum_of_max=True)),
            ("R14 splittable only", 64, dict(splittable_only=True)),
            ("R10 + R11 + R14", 112, dict(abs_starts=True, sum_of_max=True, splittable_only=True))]


@pytest.mark.parametrize("name,bits,kw", READINGS, ids=[r[0] for r in READINGS])
def test_alternative_readings_match_oracle(ns, ctx, name, bits, kw):
    """The alternative readings (flags NS_R10_ABS_STARTS, NS_R11_SUM_OF_MAX,
    NS_R14_SPLITTABLE) on both sides: column-wise searches
    identical to the oracle's beam search under the same reading, and
    ns_score_plans (fp64 and TF32x3) against the oracle's plan cost."""
    w = gen_weights(4, "mono", seed=5)
    rng = np.random.default_rng(bits)
    tasks = [small_task(rng, 14, 4) for _ in range(6)]
    for t in tasks:   # some unsplittable dims so R14 matters
        t.dims[::3] = 12
    ns.ns_load_cost_models(ctx, w)
    desc, off, caps = ns.table_descs(tasks)
    tabs = ns.ns_featurize_tables(ctx, desc, off, caps)
    out = ns.ns_shard_columnwise(ctx, tabs, 4, N=2, K=2, L=2, M=5, readings=bits)
    for i, task in enumerate(tasks):
        emb = om.TableEmbeddings(w, task)
        log = osr.DecisionLog()
        r = osr.beam_search(w, emb, task, N=2, K=2, L=2, M=5, log=log, **kw)
        exp = dict(cost=r.cost, col_plan=r.col_plan, assign=r.assign, grid_index=r.grid_index, work=r.work)
        if log.min_margin() >= RTOL:
            _compare(out, i, task, w, exp, log.min_margin(), 5)
    base = ns.ns_shard_columnwise(ctx, tabs, 4, N=2, K=2, L=2, M=5)
    # the reading changes something (the test is not vacuous)
    assert not (np.array_equal(base["cost"], out["cost"]) and np.array_equal(base["n_scores"], out["n_scores"]))
    if bits & 48:
        A = np.random.default_rng(7).integers(0, 4, size=(300, tasks[0].T)).astype(np.int8)
        emb = om.TableEmbeddings(w, tasks[0])
        tables = osr.apply_col_plan(tasks[0], [])
        ref = np.array([om.plan_cost(w, emb, tables, a.tolist(), 4, bool(bits & 16), bool(bits & 32))[0] for a in A])
        c64, _, _ = ns.ns_score_plans(ctx, tabs, 0, 4, [], A, mode=ns.NS_SCORE_FP64 | (bits & 48))
        np.testing.assert_allclose(c64, ref, rtol=1e-12)
        c32, _, _ = ns.ns_score_plans(ctx, tabs, 0, 4, [], A, mode=ns.NS_SCORE_TF32X3 | (bits & 48))
        np.testing.assert_allclose(c32, ref, rtol=1e-5)
    tabs.free()
