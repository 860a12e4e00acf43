"""Single-task C3/C4 search time with each greedy kernel selector (auto / grouped / per-lane)."""
import sys, time; sys.path.insert(0, '/root/repo')
import numpy as np, torch, paper_2305_01868_b200 as ns
from workload.synth import CONFIGS, gen_tasks, gen_weights
ctx = ns.ns_create(0)
for cfg in ("C3", "C4"):
    c = CONFIGS[cfg]; w = gen_weights(c["D"], "mono"); ns.ns_load_cost_models(ctx, w)
    task = gen_tasks(cfg, 1); d, o, cap = ns.table_descs(task)
    for greedy in (0, 1, 2):
        ts = []
        for _ in range(5):
            t0 = time.perf_counter(); tabs = ns.ns_featurize_tables(ctx, d, o, cap)
            out = ns.ns_shard_columnwise(ctx, tabs, c["D"], N=c["N"], K=c["K"], L=c["L"], M=c["M"], greedy=greedy); tabs.free(); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
        print(cfg, "greedy mode", greedy, "ms", round(1e3 * np.median(ts[1:]), 3), "cost", float(out["cost"][0]))
