"""Grouped vs per-lane greedy on the same C2 batch (must be bit-identical)."""
import sys
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_2305_01868_b200 as ns
from workload.synth import gen_tasks, gen_weights
ctx = ns.ns_create(0)
w = gen_weights(4, "mono"); ns.ns_load_cost_models(ctx, w)
tasks = gen_tasks("C2", int(sys.argv[1]))
d, o, c = ns.table_descs(tasks)
tabs = ns.ns_featurize_tables(ctx, d, o, c)
r = ns.ns_shard_tablewise(ctx, tabs, 4, M=11)
r1 = ns.ns_shard_tablewise(ctx, tabs, 4, M=11, greedy=1)
r2 = ns.ns_shard_tablewise(ctx, tabs, 4, M=11, greedy=2)
for name, x in (("auto", r), ("grouped", r1)):
    bad = np.nonzero(~((x["cost"] == r2["cost"]) | (np.isnan(x["cost"]) & np.isnan(r2["cost"]))))[0]
    print(name, "mismatches vs lanes:", len(bad), bad[:10], [ (x["cost"][i], r2["cost"][i]) for i in bad[:3]])
    bad2 = np.nonzero((x["n_scores"] != r2["n_scores"]))[0]
    print(name, "n_scores mismatches:", len(bad2))
