"""Write tests/golden/oracle_full.json: the fp64 oracle's results on the
full-size search paths (VERDICT r1 "next round" 1(b)), so the GPU tests can
compare the CUDA path's decisions with the oracle's without re-running a
minutes-long oracle on the GPU box.

Calls only oracle/ and workload/ (the seeded input recipes); nothing here
touches the CUDA path.  Each case records the oracle's (cost, column plan,
assignment, grid index, work W, column plans evaluated) and its decision log
(the smallest relative top-2 margin over every sort / greedy / grid / top-K /
global-best decision, and the number of exact ties).

    python tools/make_oracle_fixtures.py [-j 8]
"""
import argparse
import json
import math
import multiprocessing as mp
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import model as om, search as osr  # noqa: E402
from workload.synth import CONFIGS, gen_task, gen_weights  # noqa: E402

# name -> (config, task index, T override, mode, N, K, L, M, why)
CASES = {
    "C5_tw_3": ("C5", 3, None, "tablewise", 10, 3, 0, 11,
                "C5 table-wise (T = 1000, D = 128): k_build_order (T' > 256) and the wide greedy at full T"),
    "C5_tw_5": ("C5", 5, None, "tablewise", 10, 3, 0, 11, "second C5 table-wise task"),
    "C5_L1_0": ("C5", 0, None, "columnwise", 10, 3, 1, 11,
                "C5 column-wise level 1: long-list candidates (k_expand block argmax) at T' = 1000, D = 128, "
                "an oversized table forces a split"),
    "T300_D8_L2": ("C4", 0, 300, "columnwise", 10, 3, 2, 11,
                   "T = 300, D = 8, L = 2: long-list order and candidates with the grouped greedy"),
    "C3_full_0": ("C3", 0, None, "columnwise", 10, 10, 10, 11, "full C3 (K = 10, L = 10)"),
    "C3_full_1": ("C3", 1, None, "columnwise", 10, 10, 10, 11, "full C3, second task"),
    "C4_full_0": ("C4", 0, None, "columnwise", 10, 3, 10, 51, "full C4 (L = 10, M = 51 wide grid, 8 GiB cap)"),
    "C6_tw_0": ("C6", 0, None, "tablewise", 10, 3, 0, 5,
                "F4 stress: 4000 tables on 128 devices, table-wise, M = 5 (T' = 4000: k_build_order, wide greedy)"),
    "C6_L1_0": ("C6", 1, None, "columnwise", 2, 1, 1, 3,
                "F4 stress: 4000 tables on 128 devices, column-wise level 1 (N = 2, K = 1, M = 3)"),
}


def _num(x):
    return "inf" if math.isinf(x) else x


def run_case(name):
    cfg, i, T, mode, N, K, L, M, why = CASES[name]
    c = CONFIGS[cfg]
    task = gen_task(cfg, i, T=T)
    w = gen_weights(c["D"], "mono")
    t0 = time.time()
    emb = om.TableEmbeddings(w, task)
    log = osr.DecisionLog()
    if mode == "tablewise":
        r = osr.greedy_grid_search(w, emb, task, [], M, log=log)
        res = dict(cost=_num(r.cost), col_plan=[], assign=r.assign, grid_index=r.grid_index, work=r.work,
                   n_plans=1, grid_costs=[_num(x) for x in r.grid_costs])
    else:
        r = osr.beam_search(w, emb, task, N=N, K=K, L=L, M=M, log=log)
        res = dict(cost=_num(r.cost), col_plan=r.col_plan, assign=r.assign, grid_index=r.grid_index, work=r.work,
                   n_plans=r.n_plans, level_best=[_num(x) for x in r.level_best])
    kinds = sorted({k for k, _ in log.margins})
    return name, dict(config=cfg, task_index=i, T=task.T, D=c["D"], mode=mode, N=N, K=K, L=L, M=M,
                      weights="gen_weights(D, 'mono')", why=why, oracle_seconds=round(time.time() - t0, 1),
                      min_margin=_num(log.min_margin()), min_margin_by_kind={k: log.min_margin([k]) for k in kinds},
                      exact_ties=log.exact_ties, expected=res)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("-j", type=int, default=os.cpu_count())
    ap.add_argument("--only", nargs="*")
    a = ap.parse_args()
    names = a.only or list(CASES)
    # longest first
    names.sort(key=lambda n: {"C5_L1_0": 0, "C4_full_0": 1}.get(n, 2))
    with mp.Pool(min(a.j, len(names))) as pool:
        out = dict(pool.imap_unordered(run_case, names))
    path = os.path.join(ROOT, "tests", "golden", "oracle_full.json")
    old = json.load(open(path)) if os.path.exists(path) and a.only else {}
    cases = old.get("cases", {})
    cases.update(out)
    doc = {"_citation": "Written by tools/make_oracle_fixtures.py, which calls only oracle/ (fp64 GreedyGridSearch "
                        "Alg. 2 PAPER.md:289-325 and BeamSearch Alg. 1 PAPER.md:256-286, readings R1-R17 of "
                        "DESIGN.md) on workload/synth.py inputs.  No value comes from the CUDA path.",
           "cases": {k: cases[k] for k in CASES if k in cases}}
    with open(path, "w") as f:
        json.dump(doc, f, indent=1)
    for k, v in doc["cases"].items():
        print(k, v["oracle_seconds"], "s", v["expected"]["cost"], v["min_margin"], v["exact_ties"])


if __name__ == "__main__":
    main()
