"""Small runs of every hot kernel for compute-sanitizer (memcheck / racecheck /
synccheck): grouped greedy (pair-staged rows), per-lane greedy, the large-D
greedy in the 8x8 layout (k_greedy_wgrp88 with forks, k_greedy_wide88), plan
cost, precompute (both shapes), long-list orders (rank sort, merge),
score_plans in both modes (tcgen05 pooling and comm MLPs), pre-training steps, the embedding-bag kernels (hot-row backward,
exchange at one rank)."""
import sys
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_2305_01868_b200 as ns
from workload.synth import gen_task, gen_tasks, gen_weights, gen_plans
ctx = ns.ns_create(0)
w = gen_weights(4, "mono")
ns.ns_load_cost_models(ctx, w)
tasks = gen_tasks("C2", int(sys.argv[1]) if len(sys.argv) > 1 else 600)
d, o, c = ns.table_descs(tasks)
tabs = ns.ns_featurize_tables(ctx, d, o, c)
r = ns.ns_shard_tablewise(ctx, tabs, 4, M=11)                     # grouped greedy
r2 = ns.ns_shard_tablewise(ctx, tabs, 4, M=11, greedy=2)          # per-lane greedy
assert np.array_equal(r["cost"], r2["cost"])
A = gen_plans(tasks[0].T, 4, 3000, seed=1)
c64 = ns.ns_score_plans(ctx, tabs, 0, 4, [], A, mode=ns.NS_SCORE_FP64)[0]
c32 = ns.ns_score_plans(ctx, tabs, 0, 4, [], A, mode=ns.NS_SCORE_TF32X3)[0]
assert np.max(np.abs(c32 - c64) / np.abs(c64)) < 1e-5
tabs.free()
ct = [gen_task("C3", i, T=24, D=4) for i in range(4)]
d, o, c = ns.table_descs(ct)
tabs = ns.ns_featurize_tables(ctx, d, o, c)
ns.ns_shard_columnwise(ctx, tabs, 4, N=4, K=2, L=2, M=5)
tabs.free()
w40 = gen_weights(40, "mono")
ns.ns_load_cost_models(ctx, w40)
t40 = [gen_task("C3", 7, T=60, D=40)]
d, o, c = ns.table_descs(t40)
tabs = ns.ns_featurize_tables(ctx, d, o, c)
ns.ns_shard_tablewise(ctx, tabs, 40, M=3)                         # large-D greedy + BIG plan cost
g1 = ns.ns_shard_columnwise(ctx, tabs, 40, N=3, K=2, L=2, M=7, greedy=1)   # k_greedy_wgrp88 (forks)
g2 = ns.ns_shard_columnwise(ctx, tabs, 40, N=3, K=2, L=2, M=7, greedy=2)   # k_greedy_wide88
assert np.array_equal(g1["cost"], g2["cost"]) and np.array_equal(g1["assign"], g2["assign"])
tabs.free()
# long lists (T' > 256): level-0 rank sort (k_build_order), beam levels by merge (k_merge_order)
t300 = [gen_task("C3", 9, T=300, D=40), gen_task("C3", 10, T=280, D=40)]
d, o, c = ns.table_descs(t300)
tabs = ns.ns_featurize_tables(ctx, d, o, c)
m1 = ns.ns_shard_columnwise(ctx, tabs, 40, N=3, K=2, L=3, M=3)
import os
os.environ["NS_SORT_ORDERS"] = "1"
m2 = ns.ns_shard_columnwise(ctx, tabs, 40, N=3, K=2, L=3, M=3)
del os.environ["NS_SORT_ORDERS"]
assert np.array_equal(m1["cost"], m2["cost"]) and np.array_equal(m1["assign"], m2["assign"])
tabs.free()
# F2: one Adam step of each cost model
import torch
from oracle import pretrain as opt
from workload.pretrain_synth import gen_bag_indices, init_params
rng = np.random.default_rng(0)
feats = torch.from_numpy(rng.uniform(0, 1, (40, 5))).cuda()
off = torch.from_numpy(np.arange(0, 41, 4, dtype=np.int32)).cuda()
lab = torch.from_numpy(rng.uniform(1, 3, 10)).cuda()
th = torch.from_numpy(init_params(opt.COMPUTE_WIDTHS, seed=1)).cuda()
ns.ns_pretrain_compute_step(ctx, th, torch.zeros_like(th), torch.zeros_like(th), 1, 1e-3, feats, off, lab,
                            torch.arange(10, dtype=torch.int32, device="cuda"), 4)
# F3: embedding bag forward / hot-row backward / exchange (one rank)
B = 512
tabs3 = []
for rows, dim, pool, skew in ((3000, 16, 4.0, 1.5), (800, 64, 6.0, 1.8), (500, 4, 2.0, 0.0)):
    o_, i_ = gen_bag_indices(rows, pool, skew, B, rng)
    tabs3.append((torch.randn(rows, dim, device="cuda"), torch.from_numpy(i_).cuda(), torch.from_numpy(o_).cuda()))
C = 16 + 64 + 4
out = torch.zeros(B, C, device="cuda")
ns.ns_embedding_bag_forward(ctx, tabs3, B, out)
ns.ns_embedding_bag_backward_sgd(ctx, tabs3, B, torch.randn(B, C, device="cuda"), 0.01)
recv = torch.zeros(B * C, device="cuda")
ns.ns_embedding_bag_forward_exchange(ctx, tabs3, B, [C], out, recv)
ns.ns_embedding_bag_backward_exchange_sgd(ctx, tabs3, B, [C], recv, torch.zeros(B, C, device="cuda"), 0.01)
torch.cuda.synchronize()
ns.ns_destroy(ctx)
print("sanitize run ok")
