"""Single-task search latency for each BASELINE config (C1..C5), plus a sampled
oracle check of the returned plan (cost recomputed from scratch)."""
import json, sys, time
sys.path.insert(0, '/root/repo')
import numpy as np
import torch
import paper_2305_01868_b200 as ns
from workload.synth import CONFIGS, gen_tasks, gen_weights
from oracle import model as om, search as osr

ctx = ns.ns_create(0)
res = {}
for cfg in sys.argv[1:] or ["C1", "C2", "C3", "C4", "C5"]:
    c = CONFIGS[cfg]
    w = gen_weights(c["D"], "mono")
    ns.ns_load_cost_models(ctx, w)
    task = gen_tasks(cfg, 1)
    d, o, cap = ns.table_descs(task)
    times = []
    for it in range(4):
        t0 = time.perf_counter()
        tabs = ns.ns_featurize_tables(ctx, d, o, cap)
        if c["mode"] == "tablewise":
            out = ns.ns_shard_tablewise(ctx, tabs, c["D"], M=c["M"])
        else:
            out = ns.ns_shard_columnwise(ctx, tabs, c["D"], N=c["N"], K=c["K"], L=c["L"], M=c["M"])
        tabs.free()
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
    t = float(np.median(times[1:]))
    nc = int(out["n_col"][0])
    col = out["col_plan"][0, :nc].tolist() if nc else []
    tables = osr.apply_col_plan(task[0], col)
    emb = om.TableEmbeddings(w, task[0])
    a = out["assign"][0, :len(tables)].tolist()
    oc = om.plan_cost(w, emb, tables, a, c["D"])[0] if np.isfinite(out["cost"][0]) else float("inf")
    res[cfg] = {"search_ms": 1e3 * t, "scores": int(out["n_scores"][0]), "scores_per_s": int(out["n_scores"][0]) / t,
                "cost": float(out["cost"][0]), "oracle_cost_of_plan": oc, "n_col": nc}
    print(cfg, json.dumps(res[cfg]), flush=True)
ns.ns_destroy(ctx)
