import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2305_01868_b200 as ns
from workload.synth import gen_tasks, gen_weights
D = int(sys.argv[1]); mode = sys.argv[2]
ctx = ns.ns_create(0)
w = gen_weights(D, "mono")
ns.ns_load_cost_models(ctx, w)
tasks = gen_tasks("C5", 6, start=20, T=400 if D == 128 else 150, D=D)
desc, off, caps = ns.table_descs(tasks)
tabs = ns.ns_featurize_tables(ctx, desc, off, caps)
if mode == "tw":
    out = ns.ns_shard_tablewise(ctx, tabs, D, M=11, greedy=1)
else:
    out = ns.ns_shard_columnwise(ctx, tabs, D, N=4, K=2, L=3, M=11, greedy=1)
print(mode, D, out["cost"])
