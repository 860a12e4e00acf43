"""Experiment: the C5 bench step as S sub-batches on S contexts / streams
(independent tasks, concurrent kernels fill each other's level tails) vs one
context.  python tools/two_stream.py [tasks] [streams...]"""
import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2305_01868_b200 as ns
from workload.synth import gen_tasks, gen_weights
from bench import CONFIGS

c = CONFIGS["C5"]
D, N, K, L, M = c["D"], c["N"], c["K"], c["L"], c["M"]
n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
w = gen_weights(D, "mono")
tasks = gen_tasks("C5", n)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for S in [int(x) for x in sys.argv[2:]] or [1, 2]:
    streams = [torch.cuda.Stream() for _ in range(S)]
    ctxs = [ns.ns_create(0, s.cuda_stream) for s in streams]
    parts = []
    for i, ctx in enumerate(ctxs):
        ns.ns_load_cost_models(ctx, w)
        sub = tasks[i * n // S:(i + 1) * n // S]
        desc, off, caps = ns.table_descs(sub)
        T = int(np.max(np.diff(off)))
        d_desc = torch.from_numpy(desc.view(np.uint8)).cuda()
        out = dict(cost=torch.zeros(len(sub), dtype=torch.float64, device="cuda"),
                   n_col=torch.zeros(len(sub), dtype=torch.int32, device="cuda"),
                   col_plan=torch.zeros((len(sub), L), dtype=torch.int32, device="cuda"),
                   assign=torch.zeros((len(sub), T + L), dtype=torch.int8, device="cuda"),
                   grid_index=torch.zeros(len(sub), dtype=torch.int32, device="cuda"),
                   n_scores=torch.zeros(len(sub), dtype=torch.int64, device="cuda"))
        parts.append((ctx, d_desc, off, caps, out))

    def step():
        for ctx, d_desc, off, caps, out in parts:
            tabs = ns.ns_featurize_tables(ctx, d_desc, off, caps)
            ns.ns_shard_columnwise(ctx, tabs, D, N=N, K=K, L=L, M=M, out=out, async_=True)
            tabs.free()
    for _ in range(3):
        step()
    for ctx, *_ in parts:
        ns.ns_synchronize(ctx)
    W = sum(int(p[4]["n_scores"].sum()) for p in parts)
    cost = torch.cat([p[4]["cost"] for p in parts]).cpu().numpy()
    torch.cuda.synchronize()
    reps = 8
    t0 = time.perf_counter()
    for k in range(reps):
        flush.fill_(k & 0xff)
        torch.cuda.synchronize()
        step()
        for ctx, *_ in parts:
            ns.ns_synchronize(ctx)
    dt = (time.perf_counter() - t0) / reps
    free, total = torch.cuda.mem_get_info()
    print(f"[used {(total - free) / 2**30:.1f} GiB] tasks {n} streams {S}: {dt*1e3:.2f} ms/step  {W/dt:.3e} scores/s  (W {W}, cost sum {np.nansum(np.where(np.isinf(cost),0,cost)):.6e})", flush=True)
    for ctx, *_ in parts:
        ns.ns_destroy(ctx)
