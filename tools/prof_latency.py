"""Per-kernel-class device time of one single-task search (C2..C5) from the
library's event timers (ns_profile), to see where the latency goes."""
import sys
import time

sys.path.insert(0, "/root/repo")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2305_01868_b200 as ns  # noqa: E402
from workload.synth import CONFIGS, gen_tasks, gen_weights  # noqa: E402

ctx = ns.ns_create(0)
for cfg in sys.argv[1:] or ["C3", "C4", "C5"]:
    c = CONFIGS[cfg]
    w = gen_weights(c["D"], "mono")
    ns.ns_load_cost_models(ctx, w)
    task = gen_tasks(cfg, 1)
    d, o, cap = ns.table_descs(task)

    def run():
        tabs = ns.ns_featurize_tables(ctx, d, o, cap)
        if c["mode"] == "tablewise":
            ns.ns_shard_tablewise(ctx, tabs, c["D"], M=c["M"])
        else:
            ns.ns_shard_columnwise(ctx, tabs, c["D"], N=c["N"], K=c["K"], L=c["L"], M=c["M"])
        tabs.free()

    run()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    run()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    ns.ns_profile(ctx, True)
    run()
    prof = {k: ns.ns_profile_query(ctx, k) for k in ns.PROFILE_KINDS}
    ns.ns_profile(ctx, False)
    tot = sum(v[0] for v in prof.values())
    print(f"{cfg}: wall {1e3 * wall:.2f} ms, kernel sum {tot:.2f} ms: " +
          ", ".join(f"{k} {v[0]:.3f} ms/{v[1]}" for k, v in prof.items() if v[1]), flush=True)
ns.ns_destroy(ctx)
