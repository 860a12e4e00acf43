"""GPU timeline of the bench's e2e mode (pinned host descriptors in, pinned
host results out, NS_SEARCH_ASYNC), to see what the host<->device copies cost
the step: every GPU activity of the last step with its stream and gap."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from workload.synth import CONFIGS, gen_tasks, gen_weights  # noqa: E402


def main():
    import torch
    from torch.profiler import ProfilerActivity, profile
    import paper_2305_01868_b200 as ns
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
    stream = torch.cuda.current_stream()
    ctx = ns.ns_create(0, stream.cuda_stream)
    c = CONFIGS["C2"]
    w = gen_weights(c["D"], "mono")
    ns.ns_load_cost_models(ctx, w)
    tasks = gen_tasks("C2", n)
    desc, off, caps = ns.table_descs(tasks)
    T = int(np.max(np.diff(off)))
    pin = torch.from_numpy(desc.view(np.uint8)).pin_memory()
    hout = dict(cost=torch.zeros(n, dtype=torch.float64).pin_memory(), n_col=torch.zeros(n, dtype=torch.int32).pin_memory(),
                col_plan=None, assign=torch.zeros((n, T), dtype=torch.int8).pin_memory(),
                grid_index=torch.zeros(n, dtype=torch.int32).pin_memory(),
                n_scores=torch.zeros(n, dtype=torch.int64).pin_memory())

    def step():
        tabs = ns.ns_featurize_tables(ctx, pin, off, caps)
        ns.ns_shard_tablewise(ctx, tabs, c["D"], M=c["M"], out=hout, async_=True)
        tabs.free()

    for _ in range(3):
        step()
    ns.ns_synchronize(ctx)
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(4):
            step()
        ns.ns_synchronize(ctx)
    ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
    ev.sort(key=lambda e: e.time_range.start)
    starts = [i for i, e in enumerate(ev) if "k_tables_validate" in e.name]
    seg = ev[starts[-2]:starts[-1]] if len(starts) >= 2 else ev
    t0 = seg[0].time_range.start
    for e in seg:
        s, d = e.time_range.start, e.time_range.end - e.time_range.start
        print(f"{s - t0:9.1f} {d:8.1f}  {e.name[:80]}")
    per = [(ev[b].time_range.start - ev[a].time_range.start) for a, b in zip(starts, starts[1:])]
    print("step-to-step (us):", [round(p, 1) for p in per])


if __name__ == "__main__":
    main()
