#!/usr/bin/env python
"""bench.py -- NeuroShard B200 hot-path benchmark (contract: DESIGN.md §Measurement).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[1], "C2"): DLRM-style synthetic sharding tasks
of 40 tables on 4 GPUs, table-wise greedy grid search (Alg. 2, M = 11) with a
4 GiB memory cap.  One step = the whole hot path over one batch of tasks:
featurise + per-table precompute (N1), cost order, greedy placement (N4),
plan cost (N5), grid argmin (N6) -- ns_featurize_tables + ns_shard_tablewise.
Metric: candidate-plan scores per second (one score = one evaluation of
C(S_d + {t}) for a feasible device, Alg. 2's innermost unit, O(LKNMTD) of
PAPER.md:291), whole job over all ranks; tasks are partitioned over ranks
(weak scaling, no collective on the data path).

Rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

for _v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ.setdefault(_v, "1")   # the oracle baseline is timed single-threaded

import numpy as np  # noqa: E402

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from workload.synth import CONFIGS, gen_tasks, gen_weights  # noqa: E402

METRIC = "candidate plans scored/s"
CFG = "C2"
WORKLOAD = "C2: DLRM-style 40 synthetic tables on 4 GPUs, table-wise greedy grid search (M=11), 4 GiB cap"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    # 65536 tasks per step: the grouped greedy pulls column plans from a queue
    # (~22 per resident warp), so the partially filled last round is a small
    # share of the step (per-task cost 14% lower than at 16384 tasks)
    ap.add_argument("--tasks", type=int, default=65536, help="tasks per GPU per step")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--profile-run", action="store_true", help="short run for ncu (no clocks/baseline)")
    return ap.parse_args()


# --------------------------------------------------------------------------- ranks
def dist_setup(n_gpus):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        n_dev = torch.cuda.device_count()
        if n_dev >= world:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            # more ranks than GPUs (functional check of the N > 1 path on a
            # 1-GPU box): ranks share devices, NCCL refuses duplicates -> gloo
            local = local % max(n_dev, 1)
            torch.cuda.set_device(local)
            dist.init_process_group("gloo")
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def _reduce(world, x: float, op) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=op)
    return float(t.item())


def allreduce_max(world, x: float) -> float:
    """Max over ranks (the job's time is the slowest rank's)."""
    import torch.distributed as dist
    return _reduce(world, x, dist.ReduceOp.MAX) if world > 1 else x


def allreduce_sum(world, x: float) -> float:
    import torch.distributed as dist
    return _reduce(world, x, dist.ReduceOp.SUM) if world > 1 else x


def rank_tasks(cfg: str, n: int, rank: int):
    """Weak scaling: rank r owns tasks [r*n, (r+1)*n) of the config (disjoint seeds)."""
    return gen_tasks(cfg, n, start=rank * n)


# --------------------------------------------------------------------------- clocks
_REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
            0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
            0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}


class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    def __init__(self, device_index: int):
        self.samples, self.reasons, self.max_mhz = [], 0, None
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            import torch
            h = None
            try:   # match the CUDA device to the NVML device by UUID
                uuid = str(torch.cuda.get_device_properties(device_index).uuid)
                for i in range(pynvml.nvmlDeviceGetCount()):
                    hi = pynvml.nvmlDeviceGetHandleByIndex(i)
                    u = pynvml.nvmlDeviceGetUUID(hi)
                    u = u.decode() if isinstance(u, bytes) else u
                    if uuid in u:
                        h = hi
                        break
            except Exception:
                h = None
            if h is None:
                vis = os.environ.get("CUDA_VISIBLE_DEVICES")
                idx = int(vis.split(",")[device_index]) if vis and vis.split(",")[0].isdigit() else device_index
                h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.nv, self.h = pynvml, h
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover
            self.err = str(e)

    def _run(self):
        while not self.stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= int(self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
            except Exception:
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self.ok:
            self.stop = threading.Event()
            self.th = threading.Thread(target=self._run, daemon=True)
            self.th.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self.stop.set()
            self.th.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"], "samples": 0}
        names = [n for b, n in _REASONS.items() if self.reasons & b and n != "gpu_idle"]
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz, "reasons": names,
                "samples": len(self.samples)}


# --------------------------------------------------------------------------- oracle timing
def oracle_rate(tasks, w, M, budget_s):
    """Oracle GreedyGridSearch (fp64, literal head, cache off) on tasks until
    budget_s elapses; returns (scores/s, scores, seconds, tasks done)."""
    from oracle import model as om, search as osr
    t0 = time.perf_counter()
    W, done = 0, 0
    for task in tasks:
        emb = om.TableEmbeddings(w, task)
        W += osr.greedy_grid_search(w, emb, task, [], M).work
        done += 1
        if time.perf_counter() - t0 > budget_s:
            break
    dt = time.perf_counter() - t0
    return W / dt, W, dt, done


def run_reference(args, world, rank):
    """--impl reference: the oracle as it stands, timed on the host cores."""
    if rank != 0:
        return
    c = CONFIGS[CFG]
    w = gen_weights(c["D"], "mono")
    per_step = 16
    tasks = gen_tasks(CFG, per_step * (args.steps + args.warmup))
    for s in range(args.warmup):
        oracle_rate(tasks[s * per_step:(s + 1) * per_step], w, c["M"], 1e9)
    t0 = time.perf_counter()
    W = 0
    for s in range(args.warmup, args.warmup + args.steps):
        W += oracle_rate(tasks[s * per_step:(s + 1) * per_step], w, c["M"], 1e9)[1]
    dt = time.perf_counter() - t0
    v = W / dt
    cores = 1
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "scores/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD, "tasks_per_step": per_step, "parallelism": "host, 1 core"},
            "cpu_baseline": {"value": v, "unit": "scores/s", "cores": cores, "kind": "oracle",
                             "sample": f"{per_step} C2 tasks per step x {args.steps} steps (numpy fp64 oracle)"},
            "e2e": {"value": v, "unit": "scores/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- ours
def main():
    args = parse()
    import torch
    world, rank, local = dist_setup(args.gpus)
    if args.impl == "reference":
        run_reference(args, world, rank)
        return
    import paper_2305_01868_b200 as ns

    dev = local
    torch.cuda.set_device(dev)
    stream = torch.cuda.current_stream()
    ctx = ns.ns_create(dev, stream.cuda_stream)
    c = CONFIGS[CFG]
    D, M = c["D"], c["M"]
    w = gen_weights(D, "mono")
    ns.ns_load_cost_models(ctx, w)
    n = args.tasks
    tasks = rank_tasks(CFG, n, rank)          # weak scaling: own tasks per rank
    desc, off, caps = ns.table_descs(tasks)
    T = int(np.max(np.diff(off)))
    # device-resident inputs and outputs for the `value` measurement
    d_desc = torch.from_numpy(desc.view(np.uint8)).to(f"cuda:{dev}")
    dout = dict(cost=torch.zeros(n, dtype=torch.float64, device=dev), n_col=torch.zeros(n, dtype=torch.int32, device=dev),
                col_plan=None, assign=torch.zeros((n, T), dtype=torch.int8, device=dev),
                grid_index=torch.zeros(n, dtype=torch.int32, device=dev),
                n_scores=torch.zeros(n, dtype=torch.int64, device=dev))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)   # > 126 MB L2

    def step(desc_in, out):
        # NS_SEARCH_ASYNC: the call returns once the step is enqueued, so the
        # host prepares step k+1 while the GPU runs step k (results are read
        # after the synchronize that closes the timed region / the e2e step)
        tabs = ns.ns_featurize_tables(ctx, desc_in, off, caps)
        ns.ns_shard_tablewise(ctx, tabs, D, M=M, out=out, async_=True)
        tabs.free()

    for _ in range(args.warmup):
        step(d_desc, dout)
    ns.ns_synchronize(ctx)
    scores_per_step = int(dout["n_scores"].sum().item())
    n_infeasible = int(torch.isinf(dout["cost"]).sum().item())

    # ---- timed region: K steps, L2 flushed between steps (outside the events)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    # only the roofline kernel (greedy) is bracketed by events inside the timed
    # region; the per-kernel breakdown comes from a separate profiled pass
    ns.ns_profile(ctx, True, kinds=("greedy",))
    launches0 = ns.ns_kernel_launches(ctx)
    sampler = ClockSampler(dev) if not args.profile_run else None
    barrier(world)
    torch.cuda.synchronize()
    if sampler:
        sampler.__enter__()
    for k in range(args.steps):
        flush.fill_(k & 0xff)
        ev[k][0].record(stream)
        step(d_desc, dout)
        ev[k][1].record(stream)
    ns.ns_synchronize(ctx)   # also reports a deferred descriptor-validation error
    if sampler:
        sampler.__exit__()
    barrier(world)
    launches = ns.ns_kernel_launches(ctx) - launches0
    ms_steps = [a.elapsed_time(b) for a, b in ev]
    ms_local = float(np.sum(ms_steps))
    prof = {kd: ns.ns_profile_query(ctx, kd) for kd in ns.PROFILE_KINDS}
    ns.ns_profile(ctx, False)
    # per-kernel-class breakdown: the same K steps again with every class timed
    # (events around every launch; not part of the measurement)
    ns.ns_profile(ctx, True)
    for k in range(args.steps):
        flush.fill_(k & 0xff)
        step(d_desc, dout)
    ns.ns_synchronize(ctx)
    prof_all = {kd: ns.ns_profile_query(ctx, kd) for kd in ns.PROFILE_KINDS}
    ns.ns_profile(ctx, False)
    ms_total = allreduce_max(world, ms_local)
    total_scores = allreduce_sum(world, float(scores_per_step)) * args.steps
    value = total_scores / (ms_total * 1e-3)

    # ---- e2e: the same step through the public API with HOST buffers
    e2e = None
    if not args.no_e2e:
        pin_desc = torch.from_numpy(desc.view(np.uint8)).pin_memory()
        hout = dict(cost=torch.zeros(n, dtype=torch.float64).pin_memory(),
                    n_col=torch.zeros(n, dtype=torch.int32).pin_memory(), col_plan=None,
                    assign=torch.zeros((n, T), dtype=torch.int8).pin_memory(),
                    grid_index=torch.zeros(n, dtype=torch.int32).pin_memory(),
                    n_scores=torch.zeros(n, dtype=torch.int64).pin_memory())
        h2d = desc.nbytes + off.nbytes + caps.nbytes
        d2h = sum(int(v.numel() * v.element_size()) for v in hout.values() if v is not None)
        for _ in range(2):
            step(pin_desc, hout)
        ns.ns_synchronize(ctx)
        barrier(world)
        torch.cuda.synchronize()
        # K steps back to back as a user pipelining batches would run them:
        # every step copies its descriptors in from pinned host memory (on the
        # library's copy stream, overlapping the previous step's kernels) and
        # its results out to pinned host memory; one event pair on the ctx
        # stream spans all K steps (no L2 flush inside: a step's working set,
        # 335 MB of cached v rows, exceeds the 126 MB L2)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for k in range(args.steps):
            step(pin_desc, hout)
        # the last step's result copies run on the library's copy stream:
        # close the timed region only after ns_synchronize has drained both
        ns.ns_synchronize(ctx)
        b.record(stream)
        torch.cuda.synchronize()
        barrier(world)
        e_total = allreduce_max(world, float(a.elapsed_time(b)))
        assert int(hout["n_scores"].sum()) == scores_per_step
        e2e = {"value": total_scores / (e_total * 1e-3), "unit": "scores/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": e_total / args.steps,
               "mode": "K steps pipelined through the public API (NS_SEARCH_ASYNC), one event pair, "
                       "pinned host descriptors in / results out every step, no L2 flush (working set > L2)"}

    # ---- roofline of the dominant kernel (greedy, N4): FP64-pipe bound
    g_ms, g_n = prof["greedy"]
    g_avg_ms = g_ms / max(g_n, 1)
    flops_per_score = 256          # 64 x (add, max, mul, add) in fp64: DADD + DFMA on the FP64 pipe
    achieved = scores_per_step * flops_per_score / (g_avg_ms * 1e-3) / 1e12   # per launch: 1 launch / step
    clocks = sampler.summary() if sampler else {}
    sm_max = clocks.get("sm_max_mhz") or 1965
    peak = 148 * 64 * 2 * sm_max * 1e6 / 1e12     # 64 DFMA/clk/SM (tools/fp64_peak.cu measures ~59-64)
    roof = {"bound": "alu", "kernel": "k_greedy_dedup<8> (N4, grouped greedy)", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
            "frac": achieved / peak, "traffic": None, "peak_basis": "FP64 pipe: 148 SM x 64 DFMA/clk x 2 flop at "
            f"sm_max {sm_max} MHz; flops/score = 256 (64 x add, max, mul, add)",
            "greedy_ms_per_launch": g_avg_ms, "step_share": g_ms / max(ms_local, 1e-9)}
    traffic = os.path.join(ROOT, "profiles", "greedy_traffic.json")
    if os.path.exists(traffic):
        try:
            roof["traffic"] = json.load(open(traffic)).get("bytes_per_launch")
        except Exception:
            pass

    # ---- CPU baseline: the oracle on a bounded sample (rank 0, N=1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not args.profile_run:
        rate, W, dt, done = oracle_rate(gen_tasks(CFG, 2000), w, M, 12.0)
        cpu = {"value": rate, "unit": "scores/s", "cores": 1, "kind": "oracle",
               "sample": f"{done} C2 tasks ({W} scores) in {dt:.1f} s, numpy fp64, single thread"}

    # ---- secondary: single-task search latency (sharding search time per task)
    secondary = None
    if rank == 0 and not args.no_secondary and not args.profile_run:
        secondary = search_latency(ns, ctx, torch)
        secondary["score_plans"] = score_plans_rate(ns, ctx, torch)
        secondary["service"] = service_rate(ns)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "scores/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_total / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": WORKLOAD, "tasks_per_gpu": n, "tables_per_task": c["T"], "devices": D, "M": M,
                           "scores_per_step_per_gpu": scores_per_step, "infeasible_tasks": n_infeasible,
                           "weights": "random-init W-mono (paper architecture)", "parallelism": f"tasks/{world} ranks",
                           "l2": "flushed between steps (256 MiB write)"},
                "gpu_launches": int(launches), "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
                "clocks": clocks, "kernels_ms_per_step": {k: v[0] / args.steps for k, v in prof_all.items() if v[1]},
                "kernels_ms_note": "kernels_ms_per_step: a separate pass of the same K steps with CUDA events "
                                   "around every launch; roofline.greedy_ms_per_launch: events around the "
                                   "greedy only, inside the timed region",
                "secondary": secondary}
        print(json.dumps(line), flush=True)
    ns.ns_destroy(ctx)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def search_latency(ns, ctx, torch):
    """Wall time of one ns_shard_* call for ONE task (featurise included,
    model load excluded), C2 table-wise and C3 column-wise."""
    res = {}
    for cfg, mode in (("C1", "tablewise"), ("C2", "tablewise"), ("C3", "columnwise"), ("C4", "columnwise"),
                      ("C5", "columnwise")):
        c = CONFIGS[cfg]
        w = gen_weights(c["D"], "mono")
        ns.ns_load_cost_models(ctx, w)
        task = gen_tasks(cfg, 1)
        desc, off, caps = ns.table_descs(task)
        times, scores = [], 0
        for it in range(6):
            t0 = time.perf_counter()
            tabs = ns.ns_featurize_tables(ctx, desc, off, caps)
            if mode == "tablewise":
                out = ns.ns_shard_tablewise(ctx, tabs, c["D"], M=c["M"])
            else:
                out = ns.ns_shard_columnwise(ctx, tabs, c["D"], N=c["N"], K=c["K"], L=c["L"], M=c["M"])
            tabs.free()
            torch.cuda.synchronize()
            times.append(time.perf_counter() - t0)
            scores = int(out["n_scores"][0])
        t = float(np.median(times[1:]))
        res[cfg] = {"mode": mode, "search_ms_per_task": 1e3 * t, "scores": scores, "scores_per_s": scores / t}
    # batched column-wise search (multi-task batching): 64 C3
    # tasks and 4 C5 tasks per call, device time per task and scores/s
    for cfg, n in (("C3", 64), ("C5", 4)):
        c = CONFIGS[cfg]
        w = gen_weights(c["D"], "mono")
        ns.ns_load_cost_models(ctx, w)
        tasks = gen_tasks(cfg, n)
        desc, off, caps = ns.table_descs(tasks)
        times, scores = [], 0
        for it in range(3):
            t0 = time.perf_counter()
            tabs = ns.ns_featurize_tables(ctx, desc, off, caps)
            out = ns.ns_shard_columnwise(ctx, tabs, c["D"], N=c["N"], K=c["K"], L=c["L"], M=c["M"])
            tabs.free()
            torch.cuda.synchronize()
            times.append(time.perf_counter() - t0)
            scores = int(np.sum(out["n_scores"]))
        t = float(np.median(times[1:]))
        res[f"{cfg}x{n}"] = {"mode": "columnwise, batched", "tasks": n, "ms_per_task": 1e3 * t / n,
                             "scores": scores, "scores_per_s": scores / t}
    return res


def service_rate(ns):
    """the batching front end (paper_2305_01868_b200.service)
    fed by 8 submitter threads with 16384 host-side C2 tasks; wall time from
    the first submit to the last result (host packing, featurise, search and
    per-task result split included).  The bench's own long-lived objects
    (the 65536-task batches) are frozen out of the cyclic GC first, as a
    serving process would do after start-up: otherwise every gen-2
    collection triggered by the service's per-task futures walks them."""
    import gc
    import threading
    from paper_2305_01868_b200.service import ShardingService
    c = CONFIGS[CFG]
    w = gen_weights(c["D"], "mono")
    tasks = gen_tasks(CFG, 16384, start=1 << 20)
    runs = []
    with ShardingService(w, c["D"], M=c["M"], max_batch=8192, max_wait_ms=5.0) as svc:
        svc.shard(tasks[:256])   # warm-up
        gc.collect()
        gc.freeze()
        for rep in range(3):   # thread scheduling makes single runs noisy: median of 3
            b0 = svc.batches
            res = [None] * len(tasks)

            def sub(k):
                fs = [(i, svc.submit(tasks[i])) for i in range(k, len(tasks), 8)]
                for i, f in fs:
                    res[i] = f.result()

            th = [threading.Thread(target=sub, args=(k,)) for k in range(8)]
            t0 = time.perf_counter()
            for t in th:
                t.start()
            for t in th:
                t.join()
            runs.append((time.perf_counter() - t0, svc.batches - b0))
        gc.unfreeze()
    dt, batches = sorted(runs)[1]
    scores = sum(r["n_scores"] for r in res)
    return {"tasks": len(tasks), "submitters": 8, "batches": batches, "tasks_per_s": len(tasks) / dt,
            "scores_per_s": scores / dt, "ms_total": 1e3 * dt, "runs_ms": [round(1e3 * r[0], 1) for r in runs],
            "note": "median of 3 runs"}


def score_plans_rate(ns, ctx, torch):
    """ns_score_plans (the simulator as a service) on 2^20 explicit
    random plans of one C3 task (T = 80, D = 8), device-resident assignments,
    in both modes, with each stage against its own ceiling: pooling (N2) =
    T x 64 DADD + D x 64 (head) per plan on the FP64 pipe; comm MLPs (N5) =
    2 x 25856 MAC per plan on the FP64 tensor cores (DMMA, measured 37.1
    TFLOP/s, tools/fp64_peak.cu) or, split-TF32x3 on tcgen05, 3 x that on the
    TF32 tensor peak (MEASURED_PEAKS bf16 / 2)."""
    from workload.synth import gen_plans, gen_task
    c = CONFIGS["C3"]
    D = c["D"]
    w = gen_weights(D, "mono")
    ns.ns_load_cost_models(ctx, w)
    task = gen_task("C3", 0)
    desc, off, caps = ns.table_descs([task])
    tabs = ns.ns_featurize_tables(ctx, desc, off, caps)
    P = 1 << 20
    T = task.T
    A = torch.from_numpy(gen_plans(T, D, P, seed=1)).cuda()
    cost = torch.zeros(P, dtype=torch.float64, device="cuda")
    mlp_flop = 2.0 * 2 * (2 * D * 128 + 128 * 64 + 64 * 32 + 32 * 16 + 16 * D)
    pool_flop = T * 64 + D * 64 * 3
    clock = 1965e6
    fp64_pipe = 148 * 64 * clock          # DADD/s
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    tf32_peak = peaks.get("bf16_tflops", 2250.0) / 2 * 1e12
    res = {"workload": f"C3 task, T={T}, D={D}, {P} random plans (device-resident int8 assignments)"}
    for mode, name in ((ns.NS_SCORE_FP64, "fp64"), (ns.NS_SCORE_TF32X3, "tf32x3")):
        ns.ns_score_plans(ctx, tabs, 0, D, [], A, mode=mode, cost_out=cost)
        torch.cuda.synchronize()
        reps = 5
        ns.ns_profile(ctx, True)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            ns.ns_score_plans(ctx, tabs, 0, D, [], A, mode=mode, cost_out=cost)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / reps
        pool_ms = ns.ns_profile_query(ctx, "score")[0] / reps
        mlp_ms = ns.ns_profile_query(ctx, "finalize")[0] / reps
        ns.ns_profile(ctx, False)
        mlp_peak = 37.1e12 if name == "fp64" else tf32_peak
        mlp_work = mlp_flop if name == "fp64" else 3 * mlp_flop
        res[name] = {"plans_per_s": P / (ms * 1e-3), "ms_per_call": ms, "pool_ms": pool_ms, "mlp_ms": mlp_ms,
                     # pooling runs in fp64 (FP64 pipe) in fp64 mode and in fp32 (FP32
                     # pipe, 2x the lanes) in the FP32-grade TF32x3 mode
                     ("pool_frac_fp64_pipe" if name == "fp64" else "pool_frac_fp32_pipe"):
                         P * pool_flop / (pool_ms * 1e-3) / (fp64_pipe if name == "fp64" else 2 * fp64_pipe),
                     "mlp_tflops": P * mlp_work / (mlp_ms * 1e-3) / 1e12,
                     "mlp_frac": P * mlp_work / (mlp_ms * 1e-3) / mlp_peak,
                     "hbm_gbs": (P * T + P * 8) / (ms * 1e-3) / 1e9}
    tabs.free()
    return res


if __name__ == "__main__":
    main()
