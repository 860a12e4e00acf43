import numpy as np, sys
sys.path.insert(0, '/root/repo')
import paper_2305_01868_b200 as ns
from workload.synth import gen_tasks, gen_weights
ctx = ns.ns_create(0)
w = gen_weights(4, "mono"); ns.ns_load_cost_models(ctx, w)
tasks = gen_tasks("C2", 7, T=18)
d, o, c = ns.table_descs(tasks); tabs = ns.ns_featurize_tables(ctx, d, o, c)
ref = ns.ns_shard_tablewise(ctx, tabs, 4, M=11, greedy=1)
refc = ns.ns_shard_columnwise(ctx, tabs, 4, N=4, K=3, L=3, M=5, greedy=1)
ref2 = ns.ns_shard_tablewise(ctx, tabs, 4, M=11, greedy=1)
print("tablewise before/after columnwise diff", ref2["cost"] - ref["cost"])
print("repeat identical:", np.array_equal(ref["cost"], ref2["cost"]))
ns.ns_comm_init(ctx, 2, 0, None)
got = ns.ns_shard_tablewise(ctx, tabs, 4, M=11, greedy=1)
ns.ns_comm_init(ctx, 1, 0, None)
print("cost diff", got["cost"] - ref["cost"])
print("assign equal", np.array_equal(got["assign"], ref["assign"]), "grid", got["grid_index"], ref["grid_index"])
print("scores", got["n_scores"], ref["n_scores"])
del tabs
ns.ns_destroy(ctx)
print("destroyed ok")
