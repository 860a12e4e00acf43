"""Host logic of the batching front end (paper_2305_01868_b200.service,
SURVEY §8(f) F4) without a GPU: the C ABI calls are replaced by a stand-in
that records each batch and returns per-task values derived from the task, so
batch formation, result routing, column-plan slicing, error propagation and
shutdown are checked here; the GPU test test_batching_service checks the
plans themselves against a direct batched call."""
import threading

import numpy as np
import pytest

import paper_2305_01868_b200.service as S
from workload.synth import gen_task


class _Tabs:
    def free(self):
        pass


class _FakeNs:
    """ns_* stand-in: a task's 'cost' is its first table's hash size, its
    assignment the table index mod D, its column plan [T, T+1] when
    column-wise (n_col = 2)."""

    table_descs = staticmethod(S.ns.table_descs)

    def __init__(self, fail_on=None):
        self.batches = []
        self.fail_on = fail_on
        self.destroyed = False

    def ns_create(self, device):
        return 1

    def ns_load_cost_models(self, ctx, w):
        pass

    def ns_destroy(self, ctx):
        self.destroyed = True

    def ns_featurize_tables(self, ctx, desc, off, caps):
        self._desc, self._off = desc, off
        self.batches.append(len(off) - 1)
        if self.fail_on is not None and len(self.batches) == self.fail_on:
            raise RuntimeError("injected failure")
        return _Tabs()

    def _out(self, D, ncol):
        n = len(self._off) - 1
        T = np.diff(self._off)
        width = int(T.max()) + ncol
        assign = np.full((n, width), -1, dtype=np.int8)
        for i in range(n):
            assign[i, :T[i] + ncol] = np.arange(T[i] + ncol) % D
        cost = self._desc["hash_size"][self._off[:-1]].astype(np.float64)
        return {"cost": cost, "assign": assign, "grid_index": np.arange(n, dtype=np.int32) % 7,
                "n_scores": T.astype(np.int64) * D, "n_col": np.full(n, ncol, np.int32) if ncol else None,
                "col_plan": np.stack([T, T + 1], axis=1).astype(np.int32) if ncol else None}

    def ns_shard_tablewise(self, ctx, tabs, D, M, hi):
        return self._out(D, 0)

    def ns_shard_columnwise(self, ctx, tabs, D, N, K, L, M, hi):
        return self._out(D, 2)


@pytest.fixture
def fake(monkeypatch):
    f = _FakeNs()
    monkeypatch.setattr(S, "ns", f)
    return f


def _tasks(n, D=4):
    return [gen_task("C1", 1000 + i, D=D) for i in range(n)]


def _check(tasks, res, D, ncol):
    for t, r in zip(tasks, res):
        assert r["cost"] == float(t.hash[0])
        np.testing.assert_array_equal(r["assign"], np.arange(t.T + ncol) % D)
        assert r["col_plan"] == ([t.T, t.T + 1] if ncol else [])
        assert r["n_scores"] == t.T * D


@pytest.mark.parametrize("columnwise", [False, True])
def test_results_routed_to_their_tasks(fake, columnwise):
    tasks = _tasks(50)
    with S.ShardingService(None, 4, columnwise=columnwise, max_batch=16, max_wait_ms=50.0) as svc:
        res = svc.shard(tasks)
    _check(tasks, res, 4, 2 if columnwise else 0)
    assert sum(fake.batches) == 50
    assert max(fake.batches) <= 16          # max_batch respected
    assert fake.destroyed


def test_many_submitters(fake):
    tasks = _tasks(120)
    res = [None] * len(tasks)
    with S.ShardingService(None, 4, max_batch=32, max_wait_ms=2.0) as svc:
        def sub(k):
            fs = [(i, svc.submit(tasks[i])) for i in range(k, len(tasks), 4)]
            for i, f in fs:
                res[i] = f.result(timeout=30)
        th = [threading.Thread(target=sub, args=(k,)) for k in range(4)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        assert svc.tasks == 120 and svc.batches == len(fake.batches)
    _check(tasks, res, 4, 0)


def test_error_reaches_every_future_of_the_batch(monkeypatch):
    f = _FakeNs(fail_on=2)
    monkeypatch.setattr(S, "ns", f)
    tasks = _tasks(6)
    with S.ShardingService(None, 4, max_batch=3, max_wait_ms=200.0) as svc:
        first = [svc.submit(t) for t in tasks[:3]]
        assert all(x.result(timeout=30) is not None for x in first)
        second = [svc.submit(t) for t in tasks[3:]]
        for x in second:
            with pytest.raises(RuntimeError, match="injected"):
                x.result(timeout=30)
        third = svc.submit(tasks[0])              # the service keeps serving
        assert third.result(timeout=30)["cost"] == float(tasks[0].hash[0])


def test_closed_service_rejects_submits(fake):
    svc = S.ShardingService(None, 4)
    svc.close()
    with pytest.raises(RuntimeError, match="closed"):
        svc.submit(_tasks(1)[0])


def test_submit_racing_close_never_strands_a_future(fake):
    # a submit landing between the liveness check and the
    # queue put, or after the worker's final drain, must not leave a Future
    # that never resolves.  Every accepted submit resolves (result or
    # "closed" error); every rejected one raises at submit.
    tasks = _tasks(8)
    for rep in range(20):
        svc = S.ShardingService(None, 4, max_batch=4, max_wait_ms=0.5)
        accepted, stop = [], threading.Event()

        def sub():
            k = 0
            while not stop.is_set():
                try:
                    accepted.append(svc.submit(tasks[k % len(tasks)]))
                except RuntimeError:
                    return
                k += 1

        th = [threading.Thread(target=sub) for _ in range(3)]
        for t in th:
            t.start()
        svc.close()
        stop.set()
        for t in th:
            t.join()
        for f in accepted:
            try:
                f.result(timeout=10)
            except RuntimeError as e:
                assert "closed" in str(e)
