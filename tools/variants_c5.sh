# A/B: C5 single-task latency + batched C5x4 across library builds under _variants/
for v in ${VARIANTS:-w1 w4}; do cp _variants/lib_$v.so paper_2305_01868_b200/libneuroshard.so; echo "== $v"; python tools/prof_latency.py C5 2>/dev/null; python - <<'PY'
import sys, time; sys.path.insert(0, '/root/repo')
import numpy as np, torch, paper_2305_01868_b200 as ns
from workload.synth import CONFIGS, gen_tasks, gen_weights
c = CONFIGS["C5"]; ctx = ns.ns_create(0); w = gen_weights(c["D"], "mono"); ns.ns_load_cost_models(ctx, w)
tasks = gen_tasks("C5", 4); d, o, cap = ns.table_descs(tasks); ts = []
for _ in range(3):
    t0 = time.perf_counter(); tabs = ns.ns_featurize_tables(ctx, d, o, cap)
    out = ns.ns_shard_columnwise(ctx, tabs, c["D"], N=c["N"], K=c["K"], L=c["L"], M=c["M"]); tabs.free(); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
print("C5x4 batched ms/task", 1e3 * np.median(ts[1:]) / 4, "costs", [round(float(x), 6) for x in out["cost"]])
PY
done
