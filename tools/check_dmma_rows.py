import numpy as np, sys
sys.path.insert(0, '/root/repo')
import paper_2305_01868_b200 as ns
from workload.synth import gen_tasks, gen_weights, gen_plans
ctx = ns.ns_create(0)
w = gen_weights(4, "mono"); ns.ns_load_cost_models(ctx, w)
tasks = gen_tasks("C2", 1)
d, o, c = ns.table_descs(tasks); tabs = ns.ns_featurize_tables(ctx, d, o, c)
A = gen_plans(40, 4, 64, seed=3)
c1, _, _ = ns.ns_score_plans(ctx, tabs, 0, 4, [], A)
perm = np.random.default_rng(0).permutation(64)
c2, _, _ = ns.ns_score_plans(ctx, tabs, 0, 4, [], A[perm])
print("max |diff| after permutation:", np.max(np.abs(c2 - c1[perm])), "n differ", np.sum(c2 != c1[perm]))
B = np.repeat(A[:1], 64, axis=0)
c3, _, _ = ns.ns_score_plans(ctx, tabs, 0, 4, [], B)
print("identical rows identical costs:", np.all(c3 == c3[0]), np.unique(c3).size)
