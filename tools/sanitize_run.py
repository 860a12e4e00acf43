"""Small runs of every hot kernel for compute-sanitizer (memcheck / racecheck):
grouped greedy (pair-staged rows), per-lane greedy, large-D greedy, plan cost,
precompute (both shapes), score_plans in both modes (tcgen05 two tile groups)."""
import sys
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_2305_01868_b200 as ns
from workload.synth import gen_task, gen_tasks, gen_weights, gen_plans
ctx = ns.ns_create(0)
w = gen_weights(4, "mono")
ns.ns_load_cost_models(ctx, w)
tasks = gen_tasks("C2", int(sys.argv[1]) if len(sys.argv) > 1 else 600)
d, o, c = ns.table_descs(tasks)
tabs = ns.ns_featurize_tables(ctx, d, o, c)
r = ns.ns_shard_tablewise(ctx, tabs, 4, M=11)                     # grouped greedy
r2 = ns.ns_shard_tablewise(ctx, tabs, 4, M=11, greedy=2)          # per-lane greedy
assert np.array_equal(r["cost"], r2["cost"])
A = gen_plans(tasks[0].T, 4, 3000, seed=1)
c64 = ns.ns_score_plans(ctx, tabs, 0, 4, [], A, mode=ns.NS_SCORE_FP64)[0]
c32 = ns.ns_score_plans(ctx, tabs, 0, 4, [], A, mode=ns.NS_SCORE_TF32X3)[0]
assert np.max(np.abs(c32 - c64) / np.abs(c64)) < 1e-5
tabs.free()
ct = [gen_task("C3", i, T=24, D=4) for i in range(4)]
d, o, c = ns.table_descs(ct)
tabs = ns.ns_featurize_tables(ctx, d, o, c)
ns.ns_shard_columnwise(ctx, tabs, 4, N=4, K=2, L=2, M=5)
tabs.free()
w40 = gen_weights(40, "mono")
ns.ns_load_cost_models(ctx, w40)
t40 = [gen_task("C3", 7, T=60, D=40)]
d, o, c = ns.table_descs(t40)
tabs = ns.ns_featurize_tables(ctx, d, o, c)
ns.ns_shard_tablewise(ctx, tabs, 40, M=3)                         # large-D greedy + BIG plan cost
tabs.free()
ns.ns_destroy(ctx)
print("sanitize run ok")
