"""GPU timeline of bench steps (kernels, memcpys, memsets, gaps) via torch.profiler (CUPTI).

    python tools/timeline.py [--tasks 16384] [--steps 3]

Runs the bench step (featurise + async table-wise search, device-resident)
a few times and prints, for the last step, every GPU activity with its start
offset, duration and the idle gap before it -- where the step's time goes
besides the kernels.
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from workload.synth import CONFIGS, gen_tasks, gen_weights  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tasks", type=int, default=16384)
    ap.add_argument("--steps", type=int, default=3)
    args = ap.parse_args()
    import torch
    from torch.profiler import ProfilerActivity, profile

    import paper_2305_01868_b200 as ns
    stream = torch.cuda.current_stream()
    ctx = ns.ns_create(0, stream.cuda_stream)
    c = CONFIGS["C2"]
    w = gen_weights(c["D"], "mono")
    ns.ns_load_cost_models(ctx, w)
    tasks = gen_tasks("C2", args.tasks)
    desc, off, caps = ns.table_descs(tasks)
    n, T = len(tasks), int(np.max(np.diff(off)))
    d_desc = torch.from_numpy(desc.view(np.uint8)).cuda()
    dout = dict(cost=torch.zeros(n, dtype=torch.float64, device="cuda"), n_col=torch.zeros(n, dtype=torch.int32, device="cuda"),
                col_plan=None, assign=torch.zeros((n, T), dtype=torch.int8, device="cuda"),
                grid_index=torch.zeros(n, dtype=torch.int32, device="cuda"),
                n_scores=torch.zeros(n, dtype=torch.int64, device="cuda"))

    def step():
        tabs = ns.ns_featurize_tables(ctx, d_desc, off, caps)
        ns.ns_shard_tablewise(ctx, tabs, c["D"], M=c["M"], out=dout, async_=True)
        tabs.free()

    for _ in range(3):
        step()
    ns.ns_synchronize(ctx)
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(args.steps):
            step()
        ns.ns_synchronize(ctx)
    ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
    ev.sort(key=lambda e: e.time_range.start)
    # split into steps at the validate kernel (first kernel of every step)
    starts = [i for i, e in enumerate(ev) if "k_tables_validate" in e.name]
    last = ev[starts[-1]:] if starts else ev
    t0 = last[0].time_range.start
    prev_end = None
    busy = 0.0
    print(f"{'start_us':>9} {'dur_us':>8} {'gap_us':>7}  activity")
    for e in last:
        s, d = e.time_range.start, e.time_range.end - e.time_range.start
        gap = (s - prev_end) if prev_end is not None else 0.0
        prev_end = max(prev_end or 0, e.time_range.end)
        busy += d
        print(f"{s - t0:9.1f} {d:8.1f} {gap:7.1f}  {e.name[:90]}")
    span = prev_end - t0
    print(f"step span {span:.1f} us, busy {busy:.1f} us, idle {span - busy:.1f} us")
    if len(starts) >= 2:
        per = [(ev[b].time_range.start - ev[a].time_range.start) for a, b in zip(starts, starts[1:])]
        print("step-to-step (us):", [round(p, 1) for p in per])


if __name__ == "__main__":
    main()
