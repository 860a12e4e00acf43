"""Pins for oracle/model.py (O1-O6) against things other than itself:
closed forms, a hand-derived worked example, torch.nn (library routine),
invariances the paper's architecture fixes.  CPU only."""
import itertools
import math

import numpy as np
import pytest
import torch

from conftest import hand_task, hand_weights, small_task
from oracle import model as om
from oracle import search as osr
from workload.synth import gen_task, gen_weights


# ---------------------------------------------------------------- O1 closed forms
def test_featurize_closed_form():
    # dim=128 -> first component 1; hash=1e8 -> second 1.
    x = om.featurize(128, 10**8, 50.0, 2.0)
    assert x[0] == 1.0 and x[1] == 1.0 and x[2] == 1.0 and x[3] == 1.0
    # size in GiB: 2^28 rows * 1 col * 4 B = 1 GiB
    assert om.featurize(4, 1 << 28, 1.0, 0.0)[4] == 4.0
    assert om.featurize(64, 10**4, 25.0, 1.0).tolist() == [0.5, 0.5, 0.5, 0.5, 10**4 * 64 * 4 / 2**30]


# ---------------------------------------------------- O2/O3/O5 vs torch.nn (library)
def _torch_mlp(layers, relu_last):
    mods = []
    for i, (W, b) in enumerate(layers):
        lin = torch.nn.Linear(W.shape[1], W.shape[0]).double()
        with torch.no_grad():
            lin.weight.copy_(torch.from_numpy(W))
            lin.bias.copy_(torch.from_numpy(b))
        mods.append(lin)
        if i < len(layers) - 1 or relu_last:
            mods.append(torch.nn.ReLU())
    return torch.nn.Sequential(*mods)


@pytest.mark.parametrize("kind", ["mono", "signed"])
def test_mlps_match_torch_nn(kind):
    D = 8
    w = gen_weights(D, kind)
    rng = np.random.default_rng(0)
    enc_t = _torch_mlp(w.enc, True)
    head_t = _torch_mlp(w.head, False)
    fwd_t = _torch_mlp(w.comm_fwd, False)
    for _ in range(20):
        x = rng.normal(size=5)
        np.testing.assert_allclose(om.encode(w, x), enc_t(torch.from_numpy(x)).detach().numpy(),
                                   rtol=1e-13, atol=1e-14)
        s = rng.normal(size=32) * 3
        assert om.head(w, s) == pytest.approx(float(head_t(torch.from_numpy(s))), rel=1e-13, abs=1e-14)
        st, dd = rng.uniform(0, 20, D), rng.uniform(0, 1000, D)
        ref = fwd_t(torch.from_numpy(np.concatenate([st / 20.0, dd / 1024.0]))).detach().numpy()
        np.testing.assert_allclose(om.comm_costs(w.comm_fwd, st, dd, 20.0, 1024.0), ref,
                                   rtol=1e-13, atol=1e-14)


def test_zero_weights_give_bias_only():
    # zero weights -> bias-only predictions.
    D = 4
    w = gen_weights(D, "zero")
    task = gen_task("C2", 0)
    emb = om.TableEmbeddings(w, task)
    hb2 = float(w.head[1][1][0])
    for S in ([(0, int(task.dims[0]))], [(1, int(task.dims[1])), (2, int(task.dims[2]))]):
        assert om.compute_cost(w, emb, S) == hb2
    out = om.comm_costs(w.comm_fwd, np.arange(D), np.arange(D) * 7, 20.0, 1024.0)
    np.testing.assert_array_equal(out, w.comm_fwd[4][1])


def test_compute_cost_permutation_invariant():
    # "element-wise sum of all the table representations".
    w = gen_weights(4, "signed")
    task = gen_task("C2", 1)
    emb = om.TableEmbeddings(w, task)
    S = [(s, int(task.dims[s])) for s in range(6)]
    ref = om.compute_cost(w, emb, S)
    for perm in itertools.islice(itertools.permutations(S), 50):
        assert om.compute_cost(w, emb, list(perm)) == ref
    assert om.compute_cost(w, emb, []) == 0.0


# ------------------------------------------------------------ O4/O6 hand example
def test_hand_example_costs(golden_hand):
    g = golden_hand
    w, task = hand_weights(g), hand_task(g)
    emb = om.TableEmbeddings(w, task)
    tables = [(s, int(task.dims[s])) for s in range(task.T)]
    exp = g["expected"]
    for i, t in enumerate(tables):
        assert om.compute_cost(w, emb, [t]) == pytest.approx(exp["single_costs"][i], rel=1e-12)
    cost, comp, fwd, bwd, devdim = om.plan_cost(w, emb, tables, exp["assign"], task.D)
    assert cost == pytest.approx(exp["cost"], rel=1e-12)
    np.testing.assert_allclose(comp, exp["comp"], rtol=1e-12)
    np.testing.assert_allclose(fwd, exp["fwd"], rtol=1e-12)
    np.testing.assert_allclose(bwd, exp["bwd"], rtol=1e-12)
    np.testing.assert_array_equal(devdim, exp["devdim"])


# ------------------------------------------------------------------ O6 invariants
def test_plan_cost_D1_closed_form():
    # D=1 -> bottleneck = compute + fwd + bwd of the single device;
    # the forward start is 0 (comp - min comp).
    w = gen_weights(1, "mono")
    task = gen_task("C1", 0, D=1)
    emb = om.TableEmbeddings(w, task)
    tables = [(s, int(task.dims[s])) for s in range(task.T)]
    cost, comp, fwd, bwd, devdim = om.plan_cost(w, emb, tables, [0] * task.T, 1)
    dd = float(task.dims.sum())
    f = om.mlp(w.comm_fwd, np.array([0.0, dd / 1024.0]), False)[0]
    b = om.mlp(w.comm_bwd, np.array([0.0, dd / 1024.0]), False)[0]
    assert cost == comp[0] + f + b


def test_plan_cost_relabelling_invariance_inv_weights():
    # W-inv comm weights make per-device comm identical, so f is invariant
    # under device relabelling (compute model is relabelling-equivariant).
    D = 4
    w = gen_weights(D, "inv")
    task = gen_task("C2", 3)
    emb = om.TableEmbeddings(w, task)
    tables = [(s, int(task.dims[s])) for s in range(task.T)]
    rng = np.random.default_rng(5)
    for _ in range(5):
        a = rng.integers(0, D, size=task.T)
        ref = om.plan_cost(w, emb, tables, a, D)[0]
        for perm in itertools.permutations(range(D)):
            b = [perm[d] for d in a]
            assert om.plan_cost(w, emb, tables, b, D)[0] == pytest.approx(ref, rel=1e-12)


def test_plan_cost_symmetry_identical_tables():
    # identical tables split evenly -> equal per-device breakdowns.
    w = gen_weights(2, "inv")
    rng = np.random.default_rng(1)
    task = small_task(rng, 4, 2)
    task.dims[:] = 32
    task.hash[:] = 12345
    task.pooling[:] = 7.0
    task.skew[:] = 0.5
    emb = om.TableEmbeddings(w, task)
    tables = [(s, 32) for s in range(4)]
    _, comp, fwd, bwd, devdim = om.plan_cost(w, emb, tables, [0, 1, 0, 1], 2)
    assert comp[0] == comp[1] and devdim[0] == devdim[1]
    assert fwd[0] == pytest.approx(fwd[1], rel=1e-14) and bwd[0] == pytest.approx(bwd[1], rel=1e-14)


def test_plan_cost_is_max_over_devices():
    # "report the maximum cost across devices".
    w = gen_weights(4, "mono")
    task = gen_task("C2", 2)
    emb = om.TableEmbeddings(w, task)
    tables = [(s, int(task.dims[s])) for s in range(task.T)]
    a = [s % 4 for s in range(task.T)]
    cost, comp, fwd, bwd, _ = om.plan_cost(w, emb, tables, a, 4)
    assert cost == max(comp + fwd + bwd)
    assert cost > min(comp + fwd + bwd)


def test_split_conserves_dims_and_bytes():
    # PAPER.md:237 / SPEC.md:47-55: halves carry dim/2, other fields copied.
    task = gen_task("C3", 0)
    c = [0, task.T, 0, 5]
    tabs0 = osr.apply_col_plan(task, [])
    # ensure the plan is legal on this task
    legal = []
    cur = list(tabs0)
    for ci in c:
        if ci < len(cur) and cur[ci][1] % 8 == 0:
            legal.append(ci)
            cur = osr.apply_col_plan(task, legal)
    tabs = osr.apply_col_plan(task, legal)
    assert len(tabs) == task.T + len(legal)
    assert sum(d for _, d in tabs) == int(task.dims.sum())
    assert sum(osr.table_bytes(task, t) for t in tabs) == sum(osr.table_bytes(task, t) for t in tabs0)
    assert all(d % 4 == 0 for _, d in tabs)
    four = [i for i, (_, d) in enumerate(tabs0) if d % 8 != 0]
    if four:
        with pytest.raises(ValueError):
            osr.apply_col_plan(task, [four[0]])


# ---------------------------------------------------- alternative readings
def test_reduce_plan_readings():
    # R11 max of per-device sums vs the alternative sum of the
    # per-term maxima: hand values
    comp, fwd, bwd = np.array([1.0, 3.0]), np.array([5.0, 0.0]), np.array([0.0, 0.5])
    assert om.reduce_plan(comp, fwd, bwd) == 6.0
    assert om.reduce_plan(comp, fwd, bwd, sum_of_max=True) == 8.5
    # the alternative is never below the default; equal when one device dominates every term
    rng = np.random.default_rng(0)
    for _ in range(50):
        c, f, b = rng.uniform(0, 5, (3, 4))
        assert om.reduce_plan(c, f, b, True) >= om.reduce_plan(c, f, b)
    c = np.array([3.0, 1.0]); f = np.array([2.0, 1.0]); b = np.array([4.0, 0.0])
    assert om.reduce_plan(c, f, b, True) == om.reduce_plan(c, f, b) == 9.0


def test_hand_example_absolute_starts(golden_hand):
    # R10 alternative on the hand example (tests/golden/hand_example.json):
    # forward starts = comp = [3.12, 1.35] -> fwd = 0.5*start + 0.01*devdim + 1
    # = [1.56 + 0.72 + 1, 0.675 + 0.60 + 1] = [3.28, 2.275]; bwd unchanged
    # [1.864, 1.720]; cost = max(3.12 + 3.28 + 1.864, 1.35 + 2.275 + 1.72) = 8.264
    g = golden_hand
    w, task = hand_weights(g), hand_task(g)
    emb = om.TableEmbeddings(w, task)
    tables = [(s, int(task.dims[s])) for s in range(task.T)]
    cost, comp, fwd, bwd, _ = om.plan_cost(w, emb, tables, g["expected"]["assign"], 2, abs_starts=True)
    np.testing.assert_allclose(fwd, [3.28, 2.275], rtol=1e-12)
    np.testing.assert_allclose(bwd, [1.864, 1.720], rtol=1e-12)
    assert cost == pytest.approx(8.264, rel=1e-12)
    # and the sum-of-maxima reduction: 3.12 + 3.28 + 1.864 (device 0 dominates)
    assert om.plan_cost(w, emb, tables, g["expected"]["assign"], 2, True, True)[0] == pytest.approx(8.264, rel=1e-12)
