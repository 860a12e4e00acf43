"""Per-step latency of the large-D greedy kernels on an otherwise idle GPU:
one C5 task, table-wise (one column plan, 11 grid trajectories, ~1000
steps each), grouped (k_greedy_wgrp88: one chain + forks) vs per-trajectory
(k_greedy_wide88: 11 CTAs).  python tools/step_latency.py"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2305_01868_b200 as ns  # noqa: E402
from workload.synth import CONFIGS, gen_tasks, gen_weights  # noqa: E402

c = CONFIGS["C5"]
ctx = ns.ns_create(0)
ns.ns_load_cost_models(ctx, gen_weights(128, "mono"))
task = gen_tasks("C5", 1, start=3)
desc, off, caps = ns.table_descs(task)
tabs = ns.ns_featurize_tables(ctx, desc, off, caps)
for g, name in ((1, "wgrp (grouped)"), (2, "wide (per trajectory)")):
    for it in range(3):
        ns.ns_profile(ctx, True, kinds=("greedy",))
        out = ns.ns_shard_tablewise(ctx, tabs, 128, M=c["M"], greedy=g)
        ms, n = ns.ns_profile_query(ctx, "greedy")
        st = ns.ns_last_stats(ctx)
        ns.ns_profile(ctx, False)
    T = task[0].T
    print(f"{name}: greedy {ms:.3f} ms for {T} tables -> {1e3 * ms / T:.2f} us/step "
          f"({ms * 1e-3 * 1.965e9 / T:.0f} cycles/step); group_steps {st['group_steps']}", flush=True)
