"""F3 backward probe: the bench's C2 device-0 shard (batch 65536) timed with
the tables' own index skews and with skew forced to s (uniform at 0), to
separate the hot-row atomic contention from the HBM cost.
python tools/embag_probe.py [s ...]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2305_01868_b200 as ns  # noqa: E402
from workload.pretrain_synth import gen_bag_indices  # noqa: E402
from workload.synth import CONFIGS, gen_tasks, gen_weights  # noqa: E402

ctx = ns.ns_create(0)
c = CONFIGS["C2"]
ns.ns_load_cost_models(ctx, gen_weights(c["D"], "mono"))
task = gen_tasks("C2", 1, start=7)[0]
desc, off, caps = ns.table_descs([task])
tabs = ns.ns_featurize_tables(ctx, desc, off, caps)
plan = ns.ns_shard_tablewise(ctx, tabs, c["D"], M=c["M"])
mine = [k for k in range(task.T) if plan["assign"][0, k] == 0]
B = 65536


def med(fn, n=30):
    for _ in range(5):
        fn()
    ts = []
    for _ in range(n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


gen = torch.Generator("cuda").manual_seed(0)
Ws = [torch.randn((int(task.hash[k]), int(task.dims[k])), device="cuda", generator=gen).mul_(0.01) for k in mine]
C = sum(int(task.dims[k]) for k in mine)
out = torch.zeros((B, C), device="cuda")
gout = torch.randn((B, C), device="cuda", generator=gen).mul_(1e-3)
for s in [None] + [float(x) for x in sys.argv[1:]]:
    rng = np.random.default_rng(1)
    shard, dup = [], []
    for W, k in zip(Ws, mine):
        sk = float(task.skew[k]) if s is None else s
        o, i = gen_bag_indices(W.shape[0], float(task.pooling[k]), sk, B, rng)
        shard.append((W, torch.from_numpy(i).cuda(), torch.from_numpy(o).cuda()))
        # duplicates within bags and the hottest row's share
        u = sum(len(np.unique(i[o[b]:o[b + 1]])) for b in range(0, B, 64)) / max(1, o[B // 64 * 64] if False else sum(o[b + 1] - o[b] for b in range(0, B, 64)))
        hot = np.bincount(i).max() / max(1, len(i))
        dup.append((round(sk, 2), round(float(u), 3), round(float(hot), 3)))
    f = med(lambda: ns.ns_embedding_bag_forward(ctx, shard, B, out))
    b = med(lambda: ns.ns_embedding_bag_backward_sgd(ctx, shard, B, gout, 1e-4))
    print(f"skew {'own' if s is None else s}: fwd {f:.3f} ms  bwd {b:.3f} ms  (skew, unique/len in bags, hottest share) {dup}",
          flush=True)
