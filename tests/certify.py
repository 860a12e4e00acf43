"""Parity protocol for tasks with near-ties (SURVEY §8(c) "parity protocol"
rules 1-3; VERDICT r1 "next round" 1(c)).  When the oracle's decision log has
a top-2 margin below the comparison tolerance, several plans are correct and
the GPU may legitimately pick another one.  Such a plan is then checked, not
skipped:

* T8 cost parity: the returned cost equals the oracle's plan cost f of the
  returned (column plan, assignment) recomputed from scratch;
* validity: the column plan is a legal split sequence, every table is
  placed, memory caps hold (R7), and every device's dim sum is within the
  winning grid point's cap (R6, R8);
* certificate replay: re-running Alg. 2's greedy for the returned column plan
  at the returned grid point in the oracle's cost order, every device the GPU
  chose is feasible and is a tol-argmin of the oracle's scores
  C(S_d + {t}) (R5): score(chosen) <= min + tol * |min|.

Test infrastructure only (imports the oracle)."""
import math

from oracle import model as om, search as osr


def certify_plan(w, task, col_plan, assign, grid_index, cost, M, hi=1.5, tol=1e-11, emb=None, dim_cap=True):
    emb = emb or om.TableEmbeddings(w, task)
    D = task.D
    tables = osr.apply_col_plan(task, list(col_plan))      # raises on an illegal split
    assert len(assign) == len(tables)
    assert all(0 <= a < D for a in assign), "unplaced table in a feasible plan"
    # T8
    f = om.plan_cost(w, emb, tables, list(assign), D)[0]
    assert abs(cost - f) <= 1e-12 * abs(f), (cost, f)
    # validity
    sum_dim = sum(d for _, d in tables)
    cap_dim = int(math.floor(osr.grid_max_dims(sum_dim, D, M, hi)[grid_index])) if dim_cap else 10 ** 18
    load, dd = [0] * D, [0] * D
    for i, a in enumerate(assign):
        load[a] += osr.table_bytes(task, tables[i])
        dd[a] += tables[i][1]
    assert max(load) <= task.cap and max(dd) <= cap_dim
    # certificate replay in the oracle's cost order
    order = osr.cost_order(osr.single_costs(w, emb, tables))
    members = [[] for _ in range(D)]
    dsum, bsum = [0] * D, [0] * D
    for i in order:
        t = tables[i]
        bt = osr.table_bytes(task, t)
        feas = [d for d in range(D) if bsum[d] + bt <= task.cap and dsum[d] + t[1] <= cap_dim]
        a = assign[i]
        assert a in feas, f"table {i}: chosen device {a} infeasible"
        sc = {d: om.compute_cost(w, emb, members[d] + [t]) for d in feas}
        lo = min(sc.values())
        assert sc[a] <= lo + tol * abs(lo), f"table {i}: device {a} scores {sc[a]} > min {lo}"
        members[a].append(t)
        dsum[a] += t[1]
        bsum[a] += bt
    return f
