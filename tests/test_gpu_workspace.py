"""Caller-owned workspace (SURVEY §8(b) ns_set_workspace /
ns_*_workspace_bytes): a search and a plan-scoring call carve their scratch
from a torch-owned CUDA tensor of exactly the reported size and return the
same results bit for bit as with the library's own arena; one byte less is
NS_ERR_NOMEM naming the size; NULL returns to the internal arena."""
import numpy as np
import pytest

from workload.synth import gen_plans, gen_tasks, gen_weights

pytestmark = pytest.mark.gpu


def test_workspace_search_and_score():
    import torch
    import paper_2305_01868_b200 as ns
    ctx = ns.ns_create(0)
    try:
        w = gen_weights(8, "mono")
        ns.ns_load_cost_models(ctx, w)
        tasks = gen_tasks("C3", 3, T=60)
        desc, off, caps = ns.table_descs(tasks)
        tabs = ns.ns_featurize_tables(ctx, desc, off, caps)
        ref = ns.ns_shard_columnwise(ctx, tabs, 8, N=5, K=3, L=4, M=7)
        plans = gen_plans(60, 8, 5000, seed=4)
        ref_s = ns.ns_score_plans(ctx, tabs, 1, 8, [], plans)
        need = ns.ns_search_workspace_bytes(ctx, tabs.n_tasks, tabs.T_max, 8, True, N=5, K=3, L=4, M=7)
        need_s = ns.ns_score_workspace_bytes(ctx, 60, 8, 5000, False)
        assert need > 0 and need_s > 0
        buf = torch.empty(max(need, need_s), dtype=torch.uint8, device="cuda")
        ns.ns_set_workspace(ctx, buf)
        got = ns.ns_shard_columnwise(ctx, tabs, 8, N=5, K=3, L=4, M=7)
        for k in ("cost", "n_col", "col_plan", "assign", "grid_index", "n_scores"):
            assert np.array_equal(got[k], ref[k]), k
        got_s = ns.ns_score_plans(ctx, tabs, 1, 8, [], plans)
        assert np.array_equal(got_s[0], ref_s[0]) and got_s[1:] == ref_s[1:]
        # exactly the reported size suffices; one byte less is refused with the size named
        ns.ns_set_workspace(ctx, buf[:need])
        ns.ns_shard_columnwise(ctx, tabs, 8, N=5, K=3, L=4, M=7)
        ns.ns_set_workspace(ctx, torch.empty(need - 1, dtype=torch.uint8, device="cuda"))
        with pytest.raises(ns.NSError) as e:
            ns.ns_shard_columnwise(ctx, tabs, 8, N=5, K=3, L=4, M=7)
        assert e.value.status == -3 and str(need) in str(e.value)
        # back to the internal arena
        ns.ns_set_workspace(ctx, None)
        again = ns.ns_shard_columnwise(ctx, tabs, 8, N=5, K=3, L=4, M=7)
        assert np.array_equal(again["assign"], ref["assign"])
        tabs.free()
    finally:
        ns.ns_destroy(ctx)
