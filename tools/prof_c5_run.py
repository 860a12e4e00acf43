"""One C5 single-task column-wise search (for an ncu capture of k_greedy_wide88)."""
import sys
sys.path.insert(0, '/root/repo')
import torch
import paper_2305_01868_b200 as ns
from workload.synth import CONFIGS, gen_tasks, gen_weights
c = CONFIGS["C5"]
ctx = ns.ns_create(0)
w = gen_weights(c["D"], "mono")
ns.ns_load_cost_models(ctx, w)
task = gen_tasks("C5", 1)
d, o, cap = ns.table_descs(task)
for _ in range(2):
    tabs = ns.ns_featurize_tables(ctx, d, o, cap)
    ns.ns_shard_columnwise(ctx, tabs, c["D"], N=c["N"], K=c["K"], L=c["L"], M=c["M"])
    tabs.free()
torch.cuda.synchronize()
