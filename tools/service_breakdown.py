"""Host-side breakdown of the batching front end: per-stage
wall time for one batch of C2 tasks, and the service with 1 and 8 submitter
threads.  python tools/service_breakdown.py [n_tasks]"""
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2305_01868_b200 as ns  # noqa: E402
from paper_2305_01868_b200.service import ShardingService  # noqa: E402
from workload.synth import gen_weights  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
    c = bench.CONFIGS[bench.CFG]
    w = gen_weights(c["D"], "mono")
    t0 = time.perf_counter()
    tasks = bench.gen_tasks(bench.CFG, n, start=1 << 20)
    print(f"gen_tasks {1e3 * (time.perf_counter() - t0):.1f} ms")
    ctx = ns.ns_create(0)
    ns.ns_load_cost_models(ctx, w)
    for rep in range(3):
        t = {}
        t0 = time.perf_counter()
        d, o, cp = ns.table_descs(tasks)
        t["table_descs"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        tabs = ns.ns_featurize_tables(ctx, d, o, cp)
        t["featurize"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        out = ns.ns_shard_tablewise(ctx, tabs, c["D"], M=c["M"])
        t["shard"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        tabs.free()
        t["free"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        cost = out["cost"].tolist()
        assign = np.array(out["assign"], dtype=np.int8)
        r = [{"cost": cost[i], "assign": assign[i, :tasks[i].T]} for i in range(n)]
        t["split"] = time.perf_counter() - t0
        print("  ".join(f"{k} {1e3 * v:.1f} ms" for k, v in t.items()), f"(n={len(r)})")
    ns.ns_destroy(ctx)
    torch.cuda.synchronize()
    for nt in (1, 8):
        with ShardingService(w, c["D"], M=c["M"], max_batch=8192, max_wait_ms=5.0) as svc:
            svc.shard(tasks[:256])
            b0 = svc.batches
            res = [None] * n

            def sub(k):
                fs = [(i, svc.submit(tasks[i])) for i in range(k, n, nt)]
                for i, f in fs:
                    res[i] = f.result()

            th = [threading.Thread(target=sub, args=(k,)) for k in range(nt)]
            t0 = time.perf_counter()
            for x in th:
                x.start()
            for x in th:
                x.join()
            dt = time.perf_counter() - t0
            print(f"service submitters={nt}: {n / dt:.0f} tasks/s, {svc.batches - b0} batches, {1e3 * dt:.1f} ms")


if __name__ == "__main__":
    main()
