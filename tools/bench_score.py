"""ns_score_plans throughput (plans/s) for FP64 (DMMA) and TF32X3 (tcgen05) modes."""
import os, sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2305_01868_b200 as ns
from workload.synth import gen_task, gen_weights, gen_plans
ctx = ns.ns_create(0, torch.cuda.current_stream().cuda_stream)
for cfg, D in (("C2", 4), ("C3", 8)):
    w = gen_weights(D, "mono"); ns.ns_load_cost_models(ctx, w)
    task = gen_task(cfg, 0)
    d, o, c = ns.table_descs([task]); tabs = ns.ns_featurize_tables(ctx, d, o, c)
    P = 1 << 20
    A = torch.from_numpy(gen_plans(task.T, D, P, seed=1)).cuda()
    cost = torch.zeros(P, dtype=torch.float64, device="cuda")
    for mode, name, simt in ((ns.NS_SCORE_FP64, "fp64-dmma", 0), (ns.NS_SCORE_TF32X3, "tf32x3 (SIMT pooling)", 1),
                             (ns.NS_SCORE_TF32X3, "tf32x3 (tcgen05 pooling)", 0)):
        if simt:
            os.environ["NS_POOL_SIMT"] = "1"
        else:
            os.environ.pop("NS_POOL_SIMT", None)
        ns.ns_score_plans(ctx, tabs, 0, D, [], A, mode=mode, cost_out=cost)
        ns.ns_profile(ctx, True)
        torch.cuda.synchronize(); t0 = time.perf_counter()
        for _ in range(5):
            ns.ns_score_plans(ctx, tabs, 0, D, [], A, mode=mode, cost_out=cost)
        torch.cuda.synchronize(); dt = (time.perf_counter() - t0) / 5
        prof = {k: round(ns.ns_profile_query(ctx, k)[0] / 5, 3) for k in ("score", "finalize", "other")}
        ns.ns_profile(ctx, False)
        print(f"{cfg} D={D} {name}: {P/dt:.3e} plans/s  ({dt*1e3:.2f} ms per {P} plans) kernels ms {prof}", flush=True)
