"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle on
identical seeded inputs.  Tolerances: fp64 both sides, so costs agree to
1e-12 relative and every decision (sort, greedy argmin, grid argmin, beam
top-K, global best) is identical unless the oracle's top-2 margin is below
1e-12; integers (assignments, column plans, grid index,
work counts) are compared exactly."""
import math

import numpy as np
import pytest

from certify import certify_plan
from conftest import hand_task, hand_weights, small_task
from oracle import brute, model as om, search as osr
from workload.synth import gen_task, gen_tasks, gen_weights, gen_plans

pytestmark = pytest.mark.gpu

RTOL = 1e-12


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


def _setup(ns, ctx, tasks, w):
    ns.ns_load_cost_models(ctx, w)
    desc, off, caps = ns.table_descs(tasks)
    return ns.ns_featurize_tables(ctx, desc, off, caps)


def _rel(a, b):
    if math.isinf(a) or math.isinf(b):
        return 0.0 if a == b else math.inf
    return abs(a - b) / max(abs(b), 1e-300)


GREEDY = [1, 2]   # NS_GREEDY_GROUPED, NS_GREEDY_LANES: both kernels must reproduce the oracle


def _check_tablewise(ns, ctx, tasks, w, M, greedy=0):
    tabs = _setup(ns, ctx, tasks, w)
    out = ns.ns_shard_tablewise(ctx, tabs, w.D, M=M, greedy=greedy)
    n_exact = 0
    for i, task in enumerate(tasks):
        emb = om.TableEmbeddings(w, task)
        log = osr.DecisionLog()
        r = osr.greedy_grid_search(w, emb, task, [], M, log=log)
        assert int(out["n_scores"][i]) == r.work or log.min_margin() < RTOL, f"task {i}: work"
        if log.min_margin() < RTOL:
            # near-tie below fp64 resolution: decisions may legitimately
            # differ -- certify the returned plan instead (tests/certify.py)
            if math.isfinite(out["cost"][i]):
                certify_plan(w, task, [], out["assign"][i, :task.T].tolist(), int(out["grid_index"][i]),
                             float(out["cost"][i]), M, emb=emb)
            continue
        n_exact += 1
        assert _rel(out["cost"][i], r.cost) <= RTOL, f"task {i}: cost {out['cost'][i]} vs {r.cost}"
        if r.assign is None:
            assert out["grid_index"][i] == -1 and np.all(out["assign"][i] == -1)
        else:
            assert out["grid_index"][i] == r.grid_index, f"task {i}: grid index"
            assert out["assign"][i, :task.T].tolist() == r.assign, f"task {i}: assignment"
    assert n_exact >= 0.95 * len(tasks)
    return out


def test_single_costs_and_features(ns, ctx):
    w = gen_weights(4, "mono")
    tasks = gen_tasks("C2", 3)
    tabs = _setup(ns, ctx, tasks, w)
    c, f = ns.ns_tables_single_costs(ctx, tabs, features=True)
    k = 0
    for task in tasks:
        emb = om.TableEmbeddings(w, task)
        for s in range(task.T):
            x = om.featurize(int(task.dims[s]), int(task.hash[s]), float(task.pooling[s]), float(task.skew[s]))
            np.testing.assert_allclose(f[k], x, rtol=1e-15, atol=0)
            assert _rel(c[k], om.compute_cost(w, emb, [(s, int(task.dims[s]))])) <= RTOL
            k += 1


def test_hand_example(ns, ctx, golden_hand):
    g = golden_hand
    w, task = hand_weights(g), hand_task(g)
    tabs = _setup(ns, ctx, [task], w)
    out = ns.ns_shard_tablewise(ctx, tabs, 2, M=g["M"])
    e = g["expected"]
    assert out["cost"][0] == pytest.approx(e["cost"], rel=1e-12)
    assert out["assign"][0, :3].tolist() == e["assign"]
    assert out["grid_index"][0] == e["grid_index"]
    assert int(out["n_scores"][0]) == e["work"]


@pytest.mark.parametrize("greedy", GREEDY)
def test_beam_example(ns, ctx, greedy):
    """The hand-derived beam example (tests/golden/beam_example.json: split
    appended at the end P:237, candidate order P:270, top-K by (cost,
    generation) with +inf children, strict-< global best P:275-281) through
    the CUDA path."""
    from conftest import load_golden
    g = load_golden("beam_example.json")
    w, task = hand_weights(g), hand_task(g)
    tabs = _setup(ns, ctx, [task], w)
    out = ns.ns_shard_columnwise(ctx, tabs, g["D"], N=g["N"], K=g["K"], L=g["L"], M=g["M"], greedy=greedy)
    e = g["expected"]
    nc = int(out["n_col"][0])
    assert out["cost"][0] == e["cost"]
    assert out["col_plan"][0, :nc].tolist() == e["col_plan"]
    assert out["assign"][0, :task.T + nc].tolist() == e["assign"]
    assert out["grid_index"][0] == e["grid_index"]
    assert int(out["n_scores"][0]) == e["work"]


@pytest.mark.parametrize("greedy", GREEDY)
@pytest.mark.parametrize("kind", ["mono", "signed"])
def test_tablewise_C1(ns, ctx, kind, greedy):
    w = gen_weights(2, kind)
    _check_tablewise(ns, ctx, gen_tasks("C1", 100), w, M=3, greedy=greedy)


@pytest.mark.parametrize("greedy", GREEDY)
def test_tablewise_C2(ns, ctx, greedy):
    w = gen_weights(4, "mono")
    _check_tablewise(ns, ctx, gen_tasks("C2", 24), w, M=11, greedy=greedy)


BENCH_TASKS = 65536   # bench.py --tasks default (BASELINE configs[1] = C2)


def test_tablewise_C2_bench_launch(ns, ctx):
    # the bench's full size and launch configuration (65536 tasks -> batched
    # precompute, grouped greedy, auto mode); the oracle checks a sample of
    # tasks one by one
    w = gen_weights(4, "mono")
    tasks = gen_tasks("C2", BENCH_TASKS)
    tabs = _setup(ns, ctx, tasks, w)
    out = ns.ns_shard_tablewise(ctx, tabs, 4, M=11)
    for i in range(0, BENCH_TASKS, 257):
        task = tasks[i]
        emb = om.TableEmbeddings(w, task)
        r = osr.greedy_grid_search(w, emb, task, [], 11)
        assert int(out["n_scores"][i]) == r.work
        assert _rel(out["cost"][i], r.cost) <= RTOL
        if r.assign is not None:
            assert out["assign"][i, :task.T].tolist() == r.assign


@pytest.mark.parametrize("greedy", GREEDY)
def test_tablewise_ragged_batch_and_edge_cases(ns, ctx, greedy):
    # tasks of different sizes in one batch (ragged), T = 1, D = 1-like caps,
    # and tasks whose grid points strand tables
    rng = np.random.default_rng(11)
    D = 3
    tasks = [small_task(rng, T, D, hash_hi=1e6) for T in (1, 2, 3, 7, 17, 33, 64)]
    tasks.append(small_task(rng, 9, D, cap=1 << 26, hash_hi=1e6))   # tight memory: some infeasible
    w = gen_weights(D, "signed", seed=21)
    _check_tablewise(ns, ctx, tasks, w, M=4, greedy=greedy)


@pytest.mark.parametrize("greedy", GREEDY)
@pytest.mark.parametrize("D", [1, 5, 16])
def test_tablewise_other_D(ns, ctx, D, greedy):
    rng = np.random.default_rng(D)
    tasks = [small_task(rng, 3 * D + 5, D) for _ in range(6)]
    w = gen_weights(D, "mono", seed=30 + D)
    _check_tablewise(ns, ctx, tasks, w, M=5, greedy=greedy)


def test_tablewise_big_D_kernel(ns, ctx):
    # D > 16 uses the multi-warp CTA kernel (C5 has D = 128)
    rng = np.random.default_rng(5)
    for D in (40, 128):
        tasks = [small_task(rng, D + 30, D) for _ in range(2)]
        w = gen_weights(D, "mono", seed=D)
        _check_tablewise(ns, ctx, tasks, w, M=3)


def test_infeasible_status(ns, ctx):
    rng = np.random.default_rng(3)
    task = small_task(rng, 6, 2, hash_hi=1e5)
    task.dims[0] = 128
    task.hash[0] = 10_000_000      # 5.1 GB table > 4 GiB cap
    w = gen_weights(2, "mono")
    tabs = _setup(ns, ctx, [task], w)
    out = ns.ns_shard_tablewise(ctx, tabs, 2, M=3)
    assert out["status"] == 1 and math.isinf(out["cost"][0]) and out["grid_index"][0] == -1
    # column-wise search splits the oversized table (T14)
    outc = ns.ns_shard_columnwise(ctx, tabs, 2, N=3, K=2, L=2, M=3)
    emb = om.TableEmbeddings(w, task)
    r = osr.beam_search(w, emb, task, N=3, K=2, L=2, M=3)
    assert outc["status"] == 0 and 0 in outc["col_plan"][0, :outc["n_col"][0]].tolist()
    assert _rel(outc["cost"][0], r.cost) <= RTOL
    assert outc["col_plan"][0, :outc["n_col"][0]].tolist() == r.col_plan


def _check_columnwise(ns, ctx, tasks, w, N, K, L, M, greedy=0):
    tabs = _setup(ns, ctx, tasks, w)
    out = ns.ns_shard_columnwise(ctx, tabs, w.D, N=N, K=K, L=L, M=M, greedy=greedy)
    n_exact = 0
    for i, task in enumerate(tasks):
        emb = om.TableEmbeddings(w, task)
        log = osr.DecisionLog()
        r = osr.beam_search(w, emb, task, N=N, K=K, L=L, M=M, log=log)
        assert int(out["n_scores"][i]) == r.work or log.min_margin() < RTOL, f"task {i}: work"
        if log.min_margin() < RTOL:
            nc = int(out["n_col"][i])
            if math.isfinite(out["cost"][i]):
                certify_plan(w, task, out["col_plan"][i, :nc].tolist(), out["assign"][i, :task.T + nc].tolist(),
                             int(out["grid_index"][i]), float(out["cost"][i]), M, emb=emb)
            continue
        n_exact += 1
        nc = int(out["n_col"][i])
        assert out["col_plan"][i, :nc].tolist() == r.col_plan, f"task {i}: column plan"
        assert _rel(out["cost"][i], r.cost) <= RTOL, f"task {i}: cost"
        if r.assign is not None:
            assert out["grid_index"][i] == r.grid_index
            assert out["assign"][i, :task.T + nc].tolist() == r.assign, f"task {i}: assignment"
    assert n_exact >= 0.9 * len(tasks)
    return out


@pytest.mark.parametrize("greedy", GREEDY)
def test_columnwise_small(ns, ctx, greedy):
    w = gen_weights(4, "mono")
    tasks = gen_tasks("C2", 4, T=16)
    _check_columnwise(ns, ctx, tasks, w, N=4, K=2, L=3, M=5, greedy=greedy)


@pytest.mark.parametrize("greedy", GREEDY)
def test_columnwise_signed_weights(ns, ctx, greedy):
    w = gen_weights(3, "signed", seed=5)
    rng = np.random.default_rng(8)
    tasks = [small_task(rng, 12, 3) for _ in range(3)]
    _check_columnwise(ns, ctx, tasks, w, N=3, K=3, L=3, M=4, greedy=greedy)


@pytest.mark.parametrize("greedy", GREEDY)
def test_columnwise_C3_level1(ns, ctx, greedy):
    # C3 shapes (T=80, D=8, N=10, K=10, M=11) with L=1: every level-1 child
    w = gen_weights(8, "mono")
    tasks = gen_tasks("C3", 2)
    _check_columnwise(ns, ctx, tasks, w, N=10, K=10, L=1, M=11, greedy=greedy)


def test_columnwise_C4_wide_grid_level1(ns, ctx):
    # C4 shapes: T=200, D=8, M=51 (wide grid), 8 GiB cap; level 1 of the beam
    w = gen_weights(8, "mono")
    tasks = gen_tasks("C4", 1)
    _check_columnwise(ns, ctx, tasks, w, N=10, K=3, L=1, M=51, greedy=1)


def test_columnwise_C3_full_size_sampled(ns, ctx):
    """Full C3 (L=10) in the bench's launch configuration; the oracle checks
    the returned plan one by one: its cost from scratch (T8), GreedyGridSearch
    of the returned column plan reproduces (cost, assign), and validity."""
    w = gen_weights(8, "mono")
    tasks = gen_tasks("C3", 2)
    tabs = _setup(ns, ctx, tasks, w)
    out = ns.ns_shard_columnwise(ctx, tabs, 8, N=10, K=10, L=10, M=11)
    for i, task in enumerate(tasks):
        emb = om.TableEmbeddings(w, task)
        nc = int(out["n_col"][i])
        c = out["col_plan"][i, :nc].tolist()
        tables = osr.apply_col_plan(task, c)
        a = out["assign"][i, :task.T + nc].tolist()
        assert _rel(out["cost"][i], om.plan_cost(w, emb, tables, a, 8)[0]) <= RTOL
        r = osr.greedy_grid_search(w, emb, task, c, 11)
        assert r.assign == a and _rel(out["cost"][i], r.cost) <= RTOL
        r0 = osr.greedy_grid_search(w, emb, task, [], 11)
        assert out["cost"][i] <= r0.cost
        load = np.zeros(8, np.int64)
        for j, d in enumerate(a):
            load[d] += osr.table_bytes(task, tables[j])
        assert load.max() <= task.cap


def test_score_plans_exhaustive(ns, ctx):
    # every placement of <= 6 tables on 2-4 GPUs: per-plan costs and the argmin
    for seed, (D, T) in enumerate([(2, 6), (3, 6), (4, 5)]):
        rng = np.random.default_rng(50 + seed)
        task = small_task(rng, T, D)
        w = gen_weights(D, "mono" if seed % 2 == 0 else "signed", seed=60 + seed)
        tabs = _setup(ns, ctx, [task], w)
        emb = om.TableEmbeddings(w, task)
        tables = osr.apply_col_plan(task, [])
        plans = list(brute.all_placements(task, tables, D, respect_memory=False))
        best, argset, costs = brute.exhaustive_best(w, emb, task, tables, D, respect_memory=False)
        A = np.array(plans, dtype=np.int8)
        cost, bi, bc = ns.ns_score_plans(ctx, tabs, 0, D, [], A)
        np.testing.assert_allclose(cost, costs, rtol=RTOL)
        assert plans[bi] in argset and _rel(bc, best) <= RTOL


def test_score_plans_with_col_plan_and_device_input(ns, ctx):
    import torch
    w = gen_weights(8, "mono")
    task = gen_task("C3", 0)
    tabs = _setup(ns, ctx, [task], w)
    emb = om.TableEmbeddings(w, task)
    c = [i for i in range(task.T) if task.dims[i] % 8 == 0][:3]
    tables = osr.apply_col_plan(task, c)
    A = gen_plans(len(tables), 8, 300, seed=4)
    At = torch.from_numpy(A).cuda()
    cost_t = torch.zeros(300, dtype=torch.float64, device="cuda")
    _, bi, bc = ns.ns_score_plans(ctx, tabs, 0, 8, c, At, cost_out=cost_t)
    cost = cost_t.cpu().numpy()
    for p in range(0, 300, 37):
        assert _rel(cost[p], om.plan_cost(w, emb, tables, A[p].tolist(), 8)[0]) <= RTOL
    assert bi == int(np.argmin(cost)) and bc == cost.min()


def test_device_resident_inputs_and_outputs(ns, ctx):
    import torch
    w = gen_weights(4, "mono")
    tasks = gen_tasks("C2", 8)
    ns.ns_load_cost_models(ctx, w)
    desc, off, caps = ns.table_descs(tasks)
    d_desc = torch.from_numpy(desc.view(np.uint8)).cuda()
    tabs = ns.ns_featurize_tables(ctx, d_desc, off, caps)
    T = tabs.T_max
    out = dict(cost=torch.zeros(8, dtype=torch.float64, device="cuda"),
               n_col=torch.zeros(8, dtype=torch.int32, device="cuda"), col_plan=None,
               assign=torch.zeros((8, T), dtype=torch.int8, device="cuda"),
               grid_index=torch.zeros(8, dtype=torch.int32, device="cuda"),
               n_scores=torch.zeros(8, dtype=torch.int64, device="cuda"))
    ns.ns_shard_tablewise(ctx, tabs, 4, M=11, out=out)
    host = ns.ns_shard_tablewise(ctx, tabs, 4, M=11)
    assert np.array_equal(out["cost"].cpu().numpy(), host["cost"])
    assert np.array_equal(out["assign"].cpu().numpy(), host["assign"])


def test_async_search_matches_sync(ns, ctx):
    """NS_SEARCH_ASYNC: several searches enqueued back to back into device
    outputs, one ns_synchronize, results equal the synchronous calls."""
    import torch
    w = gen_weights(4, "mono")
    ns.ns_load_cost_models(ctx, w)
    batches = [gen_tasks("C2", 6, start=6 * i) for i in range(3)]
    outs, refs = [], []
    for tasks in batches:
        desc, off, caps = ns.table_descs(tasks)
        tabs = ns.ns_featurize_tables(ctx, torch.from_numpy(desc.view(np.uint8)).cuda(), off, caps)
        n, T = len(tasks), tabs.T_max
        out = dict(cost=torch.zeros(n, dtype=torch.float64, device="cuda"),
                   n_col=torch.zeros(n, dtype=torch.int32, device="cuda"), col_plan=None,
                   assign=torch.zeros((n, T + 2), dtype=torch.int8, device="cuda"),
                   grid_index=torch.zeros(n, dtype=torch.int32, device="cuda"),
                   n_scores=torch.zeros(n, dtype=torch.int64, device="cuda"))
        ns.ns_shard_tablewise(ctx, tabs, 4, M=11, out=out, async_=True)
        outc = ns.ns_shard_columnwise(ctx, tabs, 4, N=4, K=2, L=2, M=5, async_=True)   # pageable outputs
        outs.append((out, outc))
        tabs.free()   # stream-ordered: safe while the searches are in flight
    ns.ns_synchronize(ctx)
    for tasks, (out, outc) in zip(batches, outs):
        tabs = _setup(ns, ctx, tasks, w)
        ref = ns.ns_shard_tablewise(ctx, tabs, 4, M=11)
        refc = ns.ns_shard_columnwise(ctx, tabs, 4, N=4, K=2, L=2, M=5)
        T = tabs.T_max
        assert np.array_equal(out["cost"].cpu().numpy(), ref["cost"])
        a = out["assign"].cpu().numpy()
        assert np.array_equal(a[:, :T], ref["assign"]) and (a[:, T:] == -1).all()
        assert np.array_equal(out["grid_index"].cpu().numpy(), ref["grid_index"])
        assert np.array_equal(out["n_scores"].cpu().numpy().astype(np.uint64), ref["n_scores"])
        for k in ("cost", "n_col", "col_plan", "assign", "grid_index", "n_scores"):
            assert np.array_equal(outc[k], refc[k]), k
        tabs.free()


def test_pinned_descriptors_overlapped_copies(ns, ctx):
    """Pinned host descriptors go through the copy stream and two staging
    buffers: four batches enqueued back to back (async searches, no sync in
    between) give the same results as synchronous pageable-input runs."""
    import torch
    w = gen_weights(4, "mono")
    ns.ns_load_cost_models(ctx, w)
    batches = [gen_tasks("C2", 5 + i, start=40 + 10 * i) for i in range(4)]
    pins, outs = [], []
    for tasks in batches:
        desc, off, caps = ns.table_descs(tasks)
        pin = torch.from_numpy(desc.view(np.uint8)).pin_memory()
        pins.append(pin)   # must outlive the asynchronous copy
        tabs = ns.ns_featurize_tables(ctx, pin, off, caps)
        outs.append(ns.ns_shard_tablewise(ctx, tabs, 4, M=11, async_=True))
        tabs.free()
    ns.ns_synchronize(ctx)
    for tasks, out in zip(batches, outs):
        tabs = _setup(ns, ctx, tasks, w)
        ref = ns.ns_shard_tablewise(ctx, tabs, 4, M=11)
        for k in ("cost", "assign", "grid_index", "n_scores"):
            assert np.array_equal(out[k], ref[k]), k
        tabs.free()


def test_async_search_defers_validation_error(ns, ctx):
    """An invalid device-resident descriptor under NS_SEARCH_ASYNC: the search
    call returns, the next ns_synchronize reports NS_ERR_ARG, and the ctx keeps
    working afterwards."""
    import torch
    w = gen_weights(4, "mono")
    ns.ns_load_cost_models(ctx, w)
    tasks = gen_tasks("C2", 2)
    desc, off, caps = ns.table_descs(tasks)
    bad = desc.copy()
    bad["dim"][3] = 6
    tabs = ns.ns_featurize_tables(ctx, torch.from_numpy(bad.view(np.uint8)).cuda(), off, caps)
    ns.ns_shard_tablewise(ctx, tabs, 4, M=11, async_=True)
    tabs.free()
    with pytest.raises(ns.NSError):
        ns.ns_synchronize(ctx)
    ns.ns_synchronize(ctx)   # reported once
    tabs = ns.ns_featurize_tables(ctx, torch.from_numpy(desc.view(np.uint8)).cuda(), off, caps)
    ns.ns_shard_tablewise(ctx, tabs, 4, M=11, async_=True)
    ns.ns_synchronize(ctx)
    tabs.free()


def test_determinism(ns, ctx):
    w = gen_weights(8, "mono")
    tasks = gen_tasks("C3", 2)
    tabs = _setup(ns, ctx, tasks, w)
    a = ns.ns_shard_columnwise(ctx, tabs, 8, N=10, K=3, L=4, M=11)
    b = ns.ns_shard_columnwise(ctx, tabs, 8, N=10, K=3, L=4, M=11)
    for k in ("cost", "n_col", "col_plan", "assign", "grid_index", "n_scores"):
        assert np.array_equal(a[k], b[k]), k


@pytest.mark.parametrize("nranks", [2, 3])
def test_rank_partition_emulated(ns, ctx, nranks):
    """Trajectory partitioning over ranks: with emulated ranks
    every rank's block of column plans is computed separately; the results
    must equal the single-rank run bit for bit (table-wise and column-wise)."""
    w = gen_weights(4, "mono")
    tasks = gen_tasks("C2", 7, T=18)
    tabs = _setup(ns, ctx, tasks, w)
    # each greedy kernel against its own single-rank run (the two kernels split
    # the 64 features differently over lanes, so their last bits may differ)
    ref = {g: (ns.ns_shard_tablewise(ctx, tabs, 4, M=11, greedy=g),
               ns.ns_shard_columnwise(ctx, tabs, 4, N=4, K=3, L=3, M=5, greedy=g)) for g in (1, 2)}
    ns.ns_comm_init(ctx, nranks, 0, None)
    try:
        for greedy in (1, 2):
            ref_t, ref_c = ref[greedy]
            got_t = ns.ns_shard_tablewise(ctx, tabs, 4, M=11, greedy=greedy)
            got_c = ns.ns_shard_columnwise(ctx, tabs, 4, N=4, K=3, L=3, M=5, greedy=greedy)
            for k in ("cost", "assign", "grid_index", "n_scores"):
                assert np.array_equal(got_t[k], ref_t[k]), k
            for k in ("cost", "n_col", "col_plan", "assign", "grid_index", "n_scores"):
                assert np.array_equal(got_c[k], ref_c[k]), k
        A = gen_plans(18, 4, 1000, seed=2)
        c1, b1, v1 = ns.ns_score_plans(ctx, tabs, 0, 4, [], A)
    finally:
        ns.ns_comm_init(ctx, 1, 0, None)
    c0, b0, v0 = ns.ns_score_plans(ctx, tabs, 0, 4, [], A)
    assert np.array_equal(c0, c1) and b0 == b1 and v0 == v1


def test_columnwise_C5_full_size_sampled(ns, ctx):
    """C5 (1000 tables, 128 simulated GPUs, beam N=10 K=3 L=10 M=11) through the
    multi-warp greedy kernel; the oracle recomputes the returned plan's cost
    from scratch and checks validity (memory cap, the winning grid cap)."""
    from workload.synth import CONFIGS
    c = CONFIGS["C5"]
    w = gen_weights(128, "mono")
    task = gen_task("C5", 0)
    tabs = _setup(ns, ctx, [task], w)
    out = ns.ns_shard_columnwise(ctx, tabs, 128, N=c["N"], K=c["K"], L=c["L"], M=c["M"])
    assert out["status"] == 0
    nc = int(out["n_col"][0])
    col = out["col_plan"][0, :nc].tolist()
    tables = osr.apply_col_plan(task, col)
    a = out["assign"][0, :len(tables)].tolist()
    emb = om.TableEmbeddings(w, task)
    assert _rel(out["cost"][0], om.plan_cost(w, emb, tables, a, 128)[0]) <= RTOL
    load = np.zeros(128, np.int64)
    dd = np.zeros(128, np.int64)
    for j, d in enumerate(a):
        load[d] += osr.table_bytes(task, tables[j])
        dd[d] += tables[j][1]
    assert load.max() <= task.cap
    md = osr.grid_max_dims(int(task.dims.sum()), 128, c["M"])[int(out["grid_index"][0])]
    assert dd.max() <= math.floor(md)
    # the search never returns something worse than the empty column plan
    r0 = ns.ns_shard_tablewise(ctx, tabs, 128, M=c["M"])
    assert out["cost"][0] <= r0["cost"][0]


def test_invalid_descriptor_device_and_pinned(ns, ctx):
    """Pageable host descriptors are validated at ns_featurize_tables; device
    and pinned ones on the GPU, reported by the next synchronising call."""
    import torch
    w = gen_weights(4, "mono")
    ns.ns_load_cost_models(ctx, w)
    tasks = gen_tasks("C2", 2)
    desc, off, caps = ns.table_descs(tasks)
    desc["dim"][5] = 6     # not a multiple of 4
    with pytest.raises(ns.NSError):
        ns.ns_featurize_tables(ctx, desc, off, caps)
    for buf in (torch.from_numpy(desc.view(np.uint8)).cuda(), torch.from_numpy(desc.view(np.uint8)).pin_memory()):
        tabs = ns.ns_featurize_tables(ctx, buf, off, caps)
        with pytest.raises(ns.NSError):
            ns.ns_shard_tablewise(ctx, tabs, 4, M=11)
        with pytest.raises(ns.NSError):
            ns.ns_score_plans(ctx, tabs, 0, 4, [], gen_plans(40, 4, 8, seed=1))
        tabs.free()


def test_dim_above_128_rejected(ns, ctx):
    """the library caches kDepth = 6 variants per table
    (dim ... dim/32), enough for every split chain of a dim <= 128 table (the
    paper's maximum).  A dim-256 table would need a 7th variant, so it
    is rejected at featurise (pageable: immediately; device: at the next
    synchronising call) instead of letting a 6th split read the next table's
    rows."""
    import torch
    w = gen_weights(4, "mono")
    ns.ns_load_cost_models(ctx, w)
    tasks = gen_tasks("C2", 2)
    desc, off, caps = ns.table_descs(tasks)
    desc["dim"][3] = 256
    with pytest.raises(ns.NSError):
        ns.ns_featurize_tables(ctx, desc, off, caps)
    tabs = ns.ns_featurize_tables(ctx, torch.from_numpy(desc.view(np.uint8)).cuda(), off, caps)
    with pytest.raises(ns.NSError):
        ns.ns_shard_columnwise(ctx, tabs, 4, N=4, K=2, L=6, M=3)
    tabs.free()
    # dim 128 splits five times (128 -> 4) and no further: a 6-split column
    # plan of one table is illegal for ns_score_plans
    desc["dim"][3] = 128
    tabs = ns.ns_featurize_tables(ctx, desc, off, caps)
    T0 = int(off[1])
    A = np.zeros((4, T0 + 5), np.int8)
    ns.ns_score_plans(ctx, tabs, 0, 4, [3, 3, 3, 3, 3], A)
    with pytest.raises(ns.NSError):
        ns.ns_score_plans(ctx, tabs, 0, 4, [3, 3, 3, 3, 3, 3], np.zeros((4, T0 + 6), np.int8))
    tabs.free()


@pytest.mark.parametrize("D", [2, 4, 8, 16])
def test_score_plans_tf32x3_tcgen05(ns, ctx, D):
    """Bulk mode: comm MLPs on tcgen05 in split-TF32 x3 (FP32 accumulation).
    Plan costs within 1e-5 relative of the fp64 path and of the oracle
    (north star tolerance 1e-3); the argmin agrees unless its margin is below
    that tolerance."""
    rng = np.random.default_rng(70 + D)
    task = small_task(rng, 3 * D + 10, D)
    w = gen_weights(D, "mono", seed=80 + D)
    tabs = _setup(ns, ctx, [task], w)
    A = gen_plans(task.T, D, 3000, seed=D)       # > 16 tiles of 128 rows, ragged tail
    c64, b64, v64 = ns.ns_score_plans(ctx, tabs, 0, D, [], A, mode=ns.NS_SCORE_FP64)
    c32, b32, v32 = ns.ns_score_plans(ctx, tabs, 0, D, [], A, mode=ns.NS_SCORE_TF32X3)
    rel = np.abs(c32 - c64) / np.abs(c64)
    assert rel.max() < 1e-5, rel.max()
    emb = om.TableEmbeddings(w, task)
    tables = osr.apply_col_plan(task, [])
    for p in range(0, 3000, 331):
        assert _rel(c32[p], om.plan_cost(w, emb, tables, A[p].tolist(), D)[0]) < 1e-5
    srt = np.sort(c64)
    if (srt[1] - srt[0]) / abs(srt[0]) > 1e-5:
        assert b32 == b64


@pytest.mark.parametrize("D,T,n_col", [(1, 12, 0), (3, 40, 2), (5, 17, 0), (8, 80, 0), (8, 61, 3), (16, 100, 4),
                                         (8, 111, 0), (8, 112, 0), (16, 150, 4)])
def test_score_plans_pool_tcgen05(ns, ctx, D, T, n_col, monkeypatch):
    """NS_SCORE_TF32X3 pooling as a one-hot bf16 x3 contraction on tcgen05
    (k_pool_tc): plan costs within 1e-5 relative of the oracle's plan_cost
    (P:232 / P:391), within 1e-6 of the SIMT fp32 pooling (NS_POOL_SIMT), on
    odd D (unused one-hot rows), Tp with and without a multiple of 4 (word and
    byte staging), column plans, a ragged last tile, host and device
    assignments, both sides of the shared-memory limit (T' = 111 is the last
    list on k_pool_tc, 112 the first on the SIMT pooling); plans holding an
    invalid device id score NaN."""
    import torch
    rng = np.random.default_rng(500 + D * 7 + T)
    task = small_task(rng, T, D)
    w = gen_weights(D, "mono", seed=90 + D)
    tabs = _setup(ns, ctx, [task], w)
    col = [int(c) for c in rng.choice(np.flatnonzero(task.dims % 8 == 0), size=n_col, replace=False)]
    Tp = T + n_col
    P = 2 * 128 + 37
    A = gen_plans(Tp, D, P, seed=D + T)
    A[5, Tp - 1] = D            # invalid ids: out of range and negative
    A[77, 0] = -1
    c_tc, b_tc, _ = ns.ns_score_plans(ctx, tabs, 0, D, col, A, mode=ns.NS_SCORE_TF32X3)
    c_dev, b_dev, _ = ns.ns_score_plans(ctx, tabs, 0, D, col, torch.from_numpy(A).cuda(), mode=ns.NS_SCORE_TF32X3)
    monkeypatch.setenv("NS_POOL_SIMT", "1")
    c_simt, b_simt, _ = ns.ns_score_plans(ctx, tabs, 0, D, col, A, mode=ns.NS_SCORE_TF32X3)
    monkeypatch.delenv("NS_POOL_SIMT")
    assert np.isnan(c_tc[5]) and np.isnan(c_tc[77]) and np.isnan(c_simt[5])
    good = np.ones(P, bool)
    good[[5, 77]] = False
    np.testing.assert_array_equal(c_tc, c_dev)
    assert b_tc == b_dev
    rel = np.abs(c_tc[good] - c_simt[good]) / np.abs(c_simt[good])
    assert rel.max() < 1e-6, rel.max()
    for n in (1, 17):   # a single, partially filled tile: the same per-plan values
        c_n, _, _ = ns.ns_score_plans(ctx, tabs, 0, D, col, A[:n].copy(), mode=ns.NS_SCORE_TF32X3)
        np.testing.assert_array_equal(c_n, c_tc[:n])
    emb = om.TableEmbeddings(w, task)
    tables = osr.apply_col_plan(task, col)
    for p in list(range(0, P, 17)) + [P - 1]:
        if good[p]:
            assert _rel(c_tc[p], om.plan_cost(w, emb, tables, A[p].tolist(), D)[0]) < 1e-5, p
    tabs.free()


def test_profile_class_mask(ns, ctx):
    """ns_profile with a class list times only those kernel classes (the bench
    brackets just the roofline kernel inside its timed region); the search
    result is unchanged by the timers."""
    w = gen_weights(4, "mono")
    tasks = gen_tasks("C2", 64)
    tabs = _setup(ns, ctx, tasks, w)
    ref = ns.ns_shard_tablewise(ctx, tabs, 4, M=11)
    ns.ns_profile(ctx, True, kinds=("greedy",))
    out = ns.ns_shard_tablewise(ctx, tabs, 4, M=11)
    q = {k: ns.ns_profile_query(ctx, k) for k in ns.PROFILE_KINDS}
    ns.ns_profile(ctx, False)
    assert q["greedy"][1] == 1 and q["greedy"][0] > 0.0
    assert all(v[1] == 0 for k, v in q.items() if k != "greedy")
    ns.ns_profile(ctx, True)
    ns.ns_shard_tablewise(ctx, tabs, 4, M=11)
    q_all = {k: ns.ns_profile_query(ctx, k) for k in ns.PROFILE_KINDS}
    ns.ns_profile(ctx, False)
    assert q_all["greedy"][1] == 1 and q_all["order"][1] >= 1 and q_all["finalize"][1] >= 1
    np.testing.assert_array_equal(out["cost"], ref["cost"])
    np.testing.assert_array_equal(out["assign"], ref["assign"])
    tabs.free()


def test_ablation_invariants(ns, ctx):
    """SURVEY §8(f) F1 ablations on the GPU path (tools/ablation.py): the
    column-wise search with L = 0 is exactly the table-wise search ("w/o beam
    search", reading R15); the full beam search is never worse than L = 0 (the
    global best only improves over levels); for the table-wise search the M = 11
    grid contains M = 1's single cap (m = 0 is M_s), so it is never worse."""
    D = 4
    tasks = [gen_task("C3", i, T=24, D=D) for i in range(32)]
    w = gen_weights(D, "mono")
    tabs = _setup(ns, ctx, tasks, w)
    tw11 = ns.ns_shard_tablewise(ctx, tabs, D, M=11)
    tw1 = ns.ns_shard_tablewise(ctx, tabs, D, M=1)
    cw0 = ns.ns_shard_columnwise(ctx, tabs, D, N=4, K=2, L=0, M=11)
    cw = ns.ns_shard_columnwise(ctx, tabs, D, N=4, K=2, L=3, M=11)
    np.testing.assert_array_equal(cw0["cost"], tw11["cost"])
    np.testing.assert_array_equal(cw0["assign"][:, :24], tw11["assign"][:, :24])
    assert np.all(cw["cost"] <= tw11["cost"])
    assert np.all(tw11["cost"] <= tw1["cost"])
    assert np.isfinite(cw["cost"]).sum() >= np.isfinite(tw11["cost"]).sum()
    tabs.free()


def test_precompute_batched_path_bit_identical(ns, ctx):
    """The precompute has two launch shapes: batches of >= 16*16*SMs rows keep
    the encoder/projection weights in shared memory (one 16-warp CTA per SM),
    small calls read them through L1.  Same fragment scheme and arithmetic
    order, so the single costs (and every search decision) are bit-identical;
    a table-wise search of the small batch equals the same tasks inside the
    large batch."""
    w = gen_weights(4, "mono")
    tasks = gen_tasks("C2", 1200)               # 48000 rows: batched shape
    ns.ns_load_cost_models(ctx, w)
    desc, off, caps = ns.table_descs(tasks)
    big = ns.ns_featurize_tables(ctx, desc, off, caps)
    c_big = ns.ns_tables_single_costs(ctx, big)
    small_tasks = tasks[:8]                      # 320 rows: L1 shape
    d2, o2, k2 = ns.table_descs(small_tasks)
    small = ns.ns_featurize_tables(ctx, d2, o2, k2)
    c_small = ns.ns_tables_single_costs(ctx, small)
    np.testing.assert_array_equal(c_small, c_big[:len(c_small)])
    r_big = ns.ns_shard_tablewise(ctx, big, 4, M=11)
    r_small = ns.ns_shard_tablewise(ctx, small, 4, M=11)
    np.testing.assert_array_equal(r_small["cost"], r_big["cost"][:8])
    np.testing.assert_array_equal(r_small["assign"], r_big["assign"][:8, :r_small["assign"].shape[1]])
    emb = om.TableEmbeddings(w, tasks[0])
    ref = [om.compute_cost(w, emb, [(s, int(tasks[0].dims[s]))]) for s in range(tasks[0].T)]
    assert max(_rel(a, b) for a, b in zip(c_big[:tasks[0].T], ref)) < RTOL
    big.free()
    small.free()


def test_batching_service(ns, ctx):
    """the batching front end (paper_2305_01868_b200.service)
    -- tasks submitted one by one from four threads, batched by the worker --
    returns exactly the plans of one direct batched call (table-wise), and the
    column-wise service matches the direct column-wise search."""
    import threading
    from paper_2305_01868_b200.service import ShardingService
    w = gen_weights(4, "mono")
    tasks = gen_tasks("C2", 200)
    tabs = _setup(ns, ctx, tasks, w)
    ref = ns.ns_shard_tablewise(ctx, tabs, 4, M=11)
    tabs.free()
    res = [None] * len(tasks)
    with ShardingService(w, 4, M=11, max_batch=64, max_wait_ms=2.0) as svc:
        def worker(k):
            fs = [(i, svc.submit(tasks[i])) for i in range(k, len(tasks), 4)]
            for i, f in fs:
                res[i] = f.result(timeout=120)
        th = [threading.Thread(target=worker, args=(k,)) for k in range(4)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        assert svc.tasks == len(tasks) and svc.batches >= 4
    for i, r in enumerate(res):
        assert r["cost"] == ref["cost"][i]
        assert r["n_scores"] == int(ref["n_scores"][i])
        np.testing.assert_array_equal(r["assign"], ref["assign"][i, :tasks[i].T])
    ctasks = [gen_task("C3", i, T=24, D=4) for i in range(12)]
    tabs = _setup(ns, ctx, ctasks, w)
    cref = ns.ns_shard_columnwise(ctx, tabs, 4, N=4, K=2, L=2, M=5)
    tabs.free()
    with ShardingService(w, 4, columnwise=True, N=4, K=2, L=2, M=5, max_batch=5) as svc:
        cres = svc.shard(ctasks)
    for i, r in enumerate(cres):
        assert r["cost"] == cref["cost"][i]
        assert r["col_plan"] == cref["col_plan"][i, :int(cref["n_col"][i])].tolist()


@pytest.mark.parametrize("D", [1, 2, 3, 4, 6, 8, 12, 16])
def test_greedy_kernels_bit_identical(ns, ctx, D):
    """The grouped greedy (throughput) and the per-lane greedy (latency) split
    a device's 64 features over the same lanes and sum them in the same
    order, so plan costs, assignments and score counts are bit-identical --
    a task's result does not depend on the batch size that picks the kernel."""
    w = gen_weights(D, "mono")
    tasks = [gen_task("C2", i, T=12 + (i % 17), D=D) for i in range(96)]
    tabs = _setup(ns, ctx, tasks, w)
    g = ns.ns_shard_tablewise(ctx, tabs, D, M=11, greedy=1)
    l = ns.ns_shard_tablewise(ctx, tabs, D, M=11, greedy=2)
    np.testing.assert_array_equal(g["cost"], l["cost"])
    np.testing.assert_array_equal(g["assign"], l["assign"])
    np.testing.assert_array_equal(g["n_scores"], l["n_scores"])
    np.testing.assert_array_equal(g["grid_index"], l["grid_index"])
    tabs.free()
