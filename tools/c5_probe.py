"""C5 probe: batched column-wise search time and per-kernel-class breakdown
at several batch sizes (tasks per call).  Usage: python tools/c5_probe.py [n ...]"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2305_01868_b200 as ns  # noqa: E402
from workload.synth import CONFIGS, gen_tasks, gen_weights  # noqa: E402

cfg = os.environ.get("CFG", "C5")
c = CONFIGS[cfg]
ctx = ns.ns_create(0)
w = gen_weights(c["D"], "mono")
ns.ns_load_cost_models(ctx, w)
for n in [int(a) for a in sys.argv[1:]] or [1, 4, 16]:
    tasks = gen_tasks(cfg, n)
    desc, off, caps = ns.table_descs(tasks)
    for it in range(3):
        tabs = ns.ns_featurize_tables(ctx, desc, off, caps)
        if it == 2:
            ns.ns_profile(ctx, True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = ns.ns_shard_columnwise(ctx, tabs, c["D"], N=c["N"], K=c["K"], L=c["L"], M=c["M"],
                                     greedy=int(os.environ.get("GREEDY", "0")))
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        tabs.free()
    prof = {k: ns.ns_profile_query(ctx, k) for k in ns.PROFILE_KINDS}
    st = ns.ns_last_stats(ctx)
    ns.ns_profile(ctx, False)
    W = int(np.sum(out["n_scores"]))
    print(f"{cfg} n={n}: {1e3*dt:.2f} ms ({1e3*dt/n:.2f} ms/task) W={W} {W/dt:.3e} scores/s  "
          + " ".join(f"{k}={v[0]:.2f}ms/{v[1]}" for k, v in prof.items() if v[1])
          + f" | computed={st['scores_computed'] / max(W, 1):.3f}W group_steps={st['group_steps']}"
          + (f" ({st['scores_computed'] / max(st['group_steps'], 1):.1f} scores/step,"
             f" {prof['greedy'][0] * 1e-3 * 1.965e9 * 148 * 2 / max(st['group_steps'], 1):.0f} CTA-cycles/step)"
             if st['group_steps'] else ""), flush=True)
ns.ns_destroy(ctx)
