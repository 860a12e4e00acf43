"""Drive the secondary kernels once each for an ncu capture (run under ncu):
ns_score_plans TF32x3 (k_plan_mlp_tc), pre-training steps (k_pt_*),
embedding-bag forward / backward (k_bag_*)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2305_01868_b200 as ns  # noqa: E402

ctx = ns.ns_create(0)
bench.score_plans_rate(ns, ctx, torch)
bench.pretrain_rate(ns, ctx, torch)
bench.embag_rate(ns, ctx, torch)
print("done")
