"""Multi-task batching front end ("multi-task batching
service"): callers submit single sharding tasks from any thread and get a
Future; one worker thread owns an ns ctx, gathers the queued tasks into a
batch (up to ``max_batch`` tasks, or whatever arrived ``max_wait_ms`` after
the first), runs ONE featurise + search call for the batch and resolves every
caller's Future with that task's plan.

Batching is what keeps the GPU busy (a single task cannot fill 148 SMs:
DESIGN.md §12, 0.22 ms per C2 task alone vs microseconds per task in a
batch).  Results do not depend on the batch a task lands in: every task's
search is independent, and the greedy kernels chosen for small and large
batches give bit-identical plans (tests/test_gpu_parity.py).

Marshalling and threading only -- the search itself is the C ABI.
"""
from __future__ import annotations

import queue
import threading
import time
from concurrent.futures import Future
from typing import Any, List, Optional, Tuple

import numpy as np

from . import _native as ns


class ShardingService:
    """Batching search service on one GPU.

    weights: cost models (the layout ``ns_load_cost_models`` takes);
    D: devices per task (the comm models are per-D);
    columnwise: Alg. 1 + Alg. 2 (beam over column splits) instead of Alg. 2.
    A result is a dict with ``cost`` (float, +inf when infeasible),
    ``assign`` (int8 device per post-split table, -1 unplaced), ``col_plan``
    (list of split indices), ``grid_index`` and ``n_scores`` (the task's
    candidate-score count W).
    """

    def __init__(self, weights, D: int, columnwise: bool = False, N: int = 10, K: int = 3, L: int = 10,
                 M: int = 11, hi: float = 1.5, device: int = 0, max_batch: int = 4096, max_wait_ms: float = 1.0):
        self.D, self.columnwise = D, columnwise
        self.N, self.K, self.L, self.M, self.hi = N, K, L, M, hi
        self.device, self.max_batch, self.max_wait = device, max_batch, max_wait_ms * 1e-3
        self.batches = 0
        self.tasks = 0
        # SimpleQueue: C-implemented, one lock per put/get (submitters and the
        # worker share the GIL; queue.Queue's Condition bookkeeping costs more)
        self._q: "queue.SimpleQueue[Optional[Tuple[Any, Future]]]" = queue.SimpleQueue()
        self._ready = threading.Event()
        self._err: Optional[BaseException] = None
        # submit/close/worker-exit serialise on this lock: once _closed is set
        # no task can be queued behind the stop sentinel or after the drain
        self._lock = threading.Lock()
        self._closed = False
        self._worker = threading.Thread(target=self._run, args=(weights,), daemon=True)
        self._worker.start()
        self._ready.wait()
        if self._err is not None:
            raise self._err

    # ------------------------------------------------------------ public API
    def submit(self, task) -> Future:
        """Queue one task (fields dims, hash, pooling, skew, cap, T); returns
        a Future resolving to the task's plan dict."""
        f: Future = Future()
        with self._lock:
            if self._closed:
                raise RuntimeError("ShardingService is closed")
            self._q.put((task, f))
        return f

    def shard(self, tasks: List) -> List[dict]:
        """Submit several tasks and wait for all of them."""
        fs = [self.submit(t) for t in tasks]
        return [f.result() for f in fs]

    def close(self) -> None:
        with self._lock:
            if not self._closed:
                self._closed = True
                self._q.put(None)
        self._worker.join()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # ------------------------------------------------------------ worker
    def _run(self, weights) -> None:
        try:
            ctx = ns.ns_create(self.device)   # the ctx lives and dies on this thread
            ns.ns_load_cost_models(ctx, weights)
        except BaseException as e:   # pragma: no cover - reported to the constructor
            self._err = e
            with self._lock:
                self._closed = True
            self._ready.set()
            return
        self._ready.set()
        stop = False
        try:
            while not stop:
                item = self._q.get()
                if item is None:
                    break
                batch = [item]
                deadline = time.monotonic() + self.max_wait
                while len(batch) < self.max_batch:
                    left = deadline - time.monotonic()
                    if left <= 0:
                        break
                    try:
                        nxt = self._q.get(timeout=left)
                    except queue.Empty:
                        break
                    if nxt is None:
                        stop = True
                        break
                    batch.append(nxt)
                self._search(ctx, batch)
        finally:
            # no submit can pass the lock after this, so the drain below is final
            with self._lock:
                self._closed = True
            # fail whatever is still queued, then release the ctx
            while True:
                try:
                    item = self._q.get_nowait()
                except queue.Empty:
                    break
                if item is not None:
                    item[1].set_exception(RuntimeError("ShardingService closed"))
            ns.ns_destroy(ctx)

    def _search(self, ctx, batch) -> None:
        tasks = [t for t, _ in batch]
        try:
            desc, off, caps = ns.table_descs(tasks)
            tabs = ns.ns_featurize_tables(ctx, desc, off, caps)
            try:
                if self.columnwise:
                    out = ns.ns_shard_columnwise(ctx, tabs, self.D, N=self.N, K=self.K, L=self.L, M=self.M,
                                                 hi=self.hi)
                else:
                    out = ns.ns_shard_tablewise(ctx, tabs, self.D, M=self.M, hi=self.hi)
            finally:
                tabs.free()
        except BaseException as e:
            for _, f in batch:
                f.set_exception(e)
            return
        self.batches += 1
        self.tasks += len(batch)
        # one conversion per output array, then per-task views / list items
        # (the per-task host work is what bounds the service: DESIGN.md §14)
        cost = out["cost"].tolist()
        gidx = out["grid_index"].tolist()
        nsc = out["n_scores"].tolist()
        assign = np.array(out["assign"], dtype=np.int8)
        ncol = out["n_col"].tolist() if out.get("n_col") is not None else None
        colp = np.array(out["col_plan"]) if ncol is not None else None
        for i, (t, f) in enumerate(batch):
            nc = ncol[i] if ncol is not None else 0
            f.set_result({
                "cost": cost[i],
                "assign": assign[i, :t.T + nc],
                "col_plan": colp[i, :nc].tolist() if nc else [],
                "grid_index": gidx[i],
                "n_scores": nsc[i],
            })
