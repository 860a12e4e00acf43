"""ctypes binding of libneuroshard.so (include/neuroshard.h) -- marshalling only.

Every function here converts Python / numpy / torch arguments to the C ABI
and calls it; all compute happens in the CUDA library.  If the shared library
is missing the import fails loudly (there is no CPU fallback).
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Any, Optional, Sequence

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libneuroshard.so")

NS_OK, NS_INFEASIBLE = 0, 1
NS_SCORE_FP64, NS_SCORE_TF32X3 = 0, 1
_STATUS = {0: "NS_OK", 1: "NS_INFEASIBLE", -1: "NS_ERR_ARG", -2: "NS_ERR_STATE", -3: "NS_ERR_NOMEM",
           -4: "NS_ERR_CUDA", -5: "NS_ERR_NCCL", -6: "NS_ERR_INTERNAL"}

TABLE_DESC = np.dtype([("dim", "<i4"), ("reserved", "<i4"), ("hash_size", "<i8"),
                       ("pooling_factor", "<f8"), ("skew", "<f8")])
assert TABLE_DESC.itemsize == 32


class NSError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


class ns_linear(C.Structure):
    _fields_ = [("in_", C.c_int32), ("out", C.c_int32), ("W", C.POINTER(C.c_double)), ("b", C.POINTER(C.c_double))]


class ns_compute_model(C.Structure):
    _fields_ = [("enc", ns_linear * 2), ("head", ns_linear * 2)]


_ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t)
_ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_int)
_ALLTOALLV_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.POINTER(C.c_size_t), C.c_void_p,
                            C.POINTER(C.c_size_t))


class ns_host_comm(C.Structure):
    _fields_ = [("user", C.c_void_p), ("allgather", _ALLGATHER_FN), ("allreduce", _ALLREDUCE_FN),
                ("alltoallv", _ALLTOALLV_FN)]


class ns_stats(C.Structure):
    _fields_ = [("scores_computed", C.c_uint64), ("trajectories", C.c_uint64), ("group_steps", C.c_uint64),
                ("scores_linear", C.c_uint64), ("replay_rows", C.c_uint64), ("replay_reps", C.c_uint64)]


class ns_bag_table(C.Structure):
    _fields_ = [("dim", C.c_int32), ("reserved", C.c_int32), ("rows", C.c_int64), ("weights", C.c_void_p),
                ("indices", C.c_void_p), ("offsets", C.c_void_p)]


class ns_comm_model(C.Structure):
    _fields_ = [("D", C.c_int32), ("layer", ns_linear * 5), ("start_scale", C.c_double), ("dim_scale", C.c_double)]


class ns_search_params(C.Structure):
    _fields_ = [("N", C.c_int32), ("K", C.c_int32), ("L", C.c_int32), ("M", C.c_int32),
                ("grid_hi_factor", C.c_double), ("flags", C.c_uint32)]


class ns_plan_batch(C.Structure):
    _fields_ = [("cost", C.c_void_p), ("n_col", C.c_void_p), ("col_plan", C.c_void_p), ("assign", C.c_void_p),
                ("assign_stride", C.c_int32), ("grid_index", C.c_void_p), ("n_scores", C.c_void_p)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2305_01868_b200.build` "
                          "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    vp, i32, i64, u64p = C.c_void_p, C.c_int32, C.c_int64, C.POINTER(C.c_uint64)
    sig = {
        "ns_create": ([C.POINTER(vp), C.c_int, vp], C.c_int),
        "ns_destroy": ([vp], C.c_int),
        "ns_last_error": ([vp], C.c_char_p),
        "ns_set_stream": ([vp, vp], C.c_int),
        "ns_synchronize": ([vp], C.c_int),
        "ns_kernel_launches": ([vp], C.c_uint64),
        "ns_profile": ([vp, i32], C.c_int),
        "ns_profile_query": ([vp, C.c_char_p, C.POINTER(C.c_double), u64p], C.c_int),
        "ns_load_cost_models": ([vp, C.POINTER(ns_compute_model), C.POINTER(ns_comm_model),
                                 C.POINTER(ns_comm_model), u64p], C.c_int),
        "ns_featurize_tables": ([vp, vp, vp, vp, i32, C.POINTER(vp)], C.c_int),
        "ns_tables_free": ([vp], C.c_int),
        "ns_tables_single_costs": ([vp, vp, vp, vp], C.c_int),
        "ns_score_plans": ([vp, vp, i32, i32, vp, i32, vp, i64, i32, vp, C.POINTER(i64), C.POINTER(C.c_double)],
                           C.c_int),
        "ns_shard_tablewise": ([vp, vp, i32, C.POINTER(ns_search_params), C.POINTER(ns_plan_batch)], C.c_int),
        "ns_shard_columnwise": ([vp, vp, i32, C.POINTER(ns_search_params), C.POINTER(ns_plan_batch)], C.c_int),
        "ns_comm_unique_id": ([vp], C.c_int),
        "ns_comm_init": ([vp, i32, i32, vp], C.c_int),
        "ns_comm_init_host": ([vp, i32, i32, C.POINTER(ns_host_comm)], C.c_int),
        "ns_stats_query": ([vp, C.POINTER(ns_stats)], C.c_int),
        "ns_pretrain_compute_samples": ([vp, vp, i32, vp, i32, vp, vp, i32, vp, vp], C.c_int),
        "ns_pretrain_comm_samples": ([vp, vp, i32, vp, i32, i32, i64, vp, vp, vp, vp, vp, vp, i32, vp, vp, vp, vp,
                                      vp], C.c_int),
        "ns_pretrain_compute_step": ([vp, vp, vp, vp, i64, C.c_double, vp, vp, vp, vp, i32, i32, vp], C.c_int),
        "ns_pretrain_comm_step": ([vp, i32, vp, vp, vp, i64, C.c_double, vp, vp, vp, i32, vp], C.c_int),
        "ns_embedding_bag_forward": ([vp, C.POINTER(ns_bag_table), i32, i32, vp], C.c_int),
        "ns_embedding_bag_backward_sgd": ([vp, C.POINTER(ns_bag_table), i32, i32, vp, C.c_float], C.c_int),
        "ns_set_workspace": ([vp, vp, C.c_size_t], C.c_int),
        "ns_search_workspace_bytes": ([vp, i32, i32, i32, C.POINTER(ns_search_params), i32,
                                       C.POINTER(C.c_size_t)], C.c_int),
        "ns_score_workspace_bytes": ([vp, i32, i32, i64, i32, C.POINTER(C.c_size_t)], C.c_int),
        "ns_embedding_bag_forward_exchange": ([vp, C.POINTER(ns_bag_table), i32, i32, vp, vp, vp], C.c_int),
        "ns_embedding_bag_backward_exchange_sgd": ([vp, C.POINTER(ns_bag_table), i32, i32, vp, vp, vp, C.c_float],
                                                   C.c_int),
    }
    for name, (args, res) in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    return lib


LIB = _load()
EXPORTED = ["ns_create", "ns_destroy", "ns_last_error", "ns_set_stream", "ns_synchronize", "ns_kernel_launches",
            "ns_profile", "ns_profile_query",
            "ns_load_cost_models", "ns_featurize_tables", "ns_tables_free", "ns_tables_single_costs",
            "ns_score_plans", "ns_shard_tablewise", "ns_shard_columnwise", "ns_comm_unique_id", "ns_comm_init",
            "ns_comm_init_host", "ns_stats_query", "ns_pretrain_compute_samples", "ns_pretrain_comm_samples",
            "ns_pretrain_compute_step", "ns_pretrain_comm_step", "ns_embedding_bag_forward",
            "ns_embedding_bag_backward_sgd", "ns_embedding_bag_forward_exchange",
            "ns_embedding_bag_backward_exchange_sgd", "ns_set_workspace", "ns_search_workspace_bytes",
            "ns_score_workspace_bytes"]


def _check(ctx, status: int, allow_infeasible: bool = True) -> int:
    if status < 0:
        msg = LIB.ns_last_error(ctx).decode() if ctx else ""
        raise NSError(status, msg)
    if status == NS_INFEASIBLE and not allow_infeasible:
        raise NSError(status, "infeasible")
    return status


def _ptr(x: Any) -> Optional[int]:
    """Host numpy array or torch tensor (host or CUDA) -> raw address."""
    if x is None:
        return None
    if isinstance(x, np.ndarray):
        assert x.flags["C_CONTIGUOUS"], "arrays must be C-contiguous"
        return x.ctypes.data
    if hasattr(x, "data_ptr"):
        assert x.is_contiguous(), "tensors must be contiguous"
        return x.data_ptr()
    raise TypeError(type(x))


# ----------------------------------------------------------------- lifecycle
def ns_create(device: int = 0, stream: Optional[int] = None) -> int:
    h = C.c_void_p()
    _check(None, LIB.ns_create(C.byref(h), device, stream))
    _LIVE_CTX.add(h.value)
    return h.value


_LIVE_CTX: set = set()


def ns_destroy(ctx: int) -> None:
    """Destroys the ctx and every ns_tables still owned by it."""
    _LIVE_CTX.discard(ctx)
    _check(ctx, LIB.ns_destroy(ctx))


def ns_set_stream(ctx: int, stream: Optional[int]) -> None:
    _check(ctx, LIB.ns_set_stream(ctx, stream))


def ns_synchronize(ctx: int) -> None:
    _check(ctx, LIB.ns_synchronize(ctx))


def ns_kernel_launches(ctx: int) -> int:
    return int(LIB.ns_kernel_launches(ctx))


def ns_profile(ctx: int, enable: bool, kinds=None) -> None:
    """Kernel timers on/off; kinds = iterable of PROFILE_KINDS names to time
    only those classes (fewer events inside a timed region)."""
    mode = 1 if enable else 0
    if enable and kinds is not None:
        mode = 0
        for k in kinds:
            mode |= 1 << (PROFILE_KINDS.index(k) + 1)
    _check(ctx, LIB.ns_profile(ctx, mode))


def ns_last_stats(ctx: int) -> dict:
    """Work counters since the last ns_profile call (ns_stats_query)."""
    st = ns_stats()
    _check(ctx, LIB.ns_stats_query(ctx, C.byref(st)))
    return {"scores_computed": int(st.scores_computed), "trajectories": int(st.trajectories),
            "group_steps": int(st.group_steps), "scores_linear": int(st.scores_linear),
            "replay_rows": int(st.replay_rows), "replay_reps": int(st.replay_reps)}


PROFILE_KINDS = ("precompute", "validate", "order", "expand", "greedy", "finalize", "select", "score", "other")


def ns_profile_query(ctx: int, kernel: str):
    """(total device ms, launches) of one kernel class since ns_profile."""
    ms, n = C.c_double(), C.c_uint64()
    _check(ctx, LIB.ns_profile_query(ctx, kernel.encode(), C.byref(ms), C.byref(n)))
    return ms.value, n.value


# ----------------------------------------------------------------- models
def _lin(W: np.ndarray, b: np.ndarray, keep: list) -> ns_linear:
    W = np.ascontiguousarray(W, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64).reshape(-1)
    keep += [W, b]
    return ns_linear(W.shape[1], W.shape[0], W.ctypes.data_as(C.POINTER(C.c_double)),
                     b.ctypes.data_as(C.POINTER(C.c_double)))


def ns_load_cost_models(ctx: int, weights) -> int:
    """weights: object with .enc, .head, .comm_fwd, .comm_bwd (lists of (W, b)),
    .D, .start_scale, .dim_scale (see workload.synth.Weights).  Returns the
    fingerprint."""
    keep: list = []
    cm = ns_compute_model()
    for i in range(2):
        cm.enc[i] = _lin(*weights.enc[i], keep)
        cm.head[i] = _lin(*weights.head[i], keep)
    comms = []
    for layers in (weights.comm_fwd, weights.comm_bwd):
        m = ns_comm_model()
        m.D = weights.D
        for i in range(5):
            m.layer[i] = _lin(*layers[i], keep)
        m.start_scale = weights.start_scale
        m.dim_scale = weights.dim_scale
        comms.append(m)
    fp = C.c_uint64()
    _check(ctx, LIB.ns_load_cost_models(ctx, C.byref(cm), C.byref(comms[0]), C.byref(comms[1]), C.byref(fp)))
    return fp.value


# ----------------------------------------------------------------- tables
def table_descs(tasks: Sequence) -> tuple:
    """Pack tasks (objects with dims/hash/pooling/skew/cap) into the ABI's
    descriptor array, offsets and caps (host numpy)."""
    off = np.zeros(len(tasks) + 1, dtype=np.int32)
    np.cumsum([t.T for t in tasks], out=off[1:])
    caps = np.fromiter((t.cap for t in tasks), dtype=np.int64, count=len(tasks))
    desc = np.zeros(int(off[-1]), dtype=TABLE_DESC)
    if len(tasks):
        desc["dim"] = np.concatenate([t.dims for t in tasks])
        desc["hash_size"] = np.concatenate([t.hash for t in tasks])
        desc["pooling_factor"] = np.concatenate([t.pooling for t in tasks])
        desc["skew"] = np.concatenate([t.skew for t in tasks])
    return desc, off, caps


class Tables:
    """Owning handle of an ns_tables batch."""

    def __init__(self, ctx: int, handle: int, offsets: np.ndarray, T_max: int):
        self.ctx, self.handle, self.offsets, self.T_max = ctx, handle, offsets, T_max
        self.n_tasks = len(offsets) - 1

    def free(self):
        if self.handle and self.ctx in _LIVE_CTX:   # ns_destroy already freed it otherwise
            LIB.ns_tables_free(self.handle)
        self.handle = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def ns_featurize_tables(ctx: int, desc, offsets: np.ndarray, caps: np.ndarray) -> Tables:
    """desc: TABLE_DESC numpy array (host) or a CUDA uint8 tensor holding the
    same bytes; offsets/caps host numpy."""
    offsets = np.ascontiguousarray(offsets, dtype=np.int32)
    caps = np.ascontiguousarray(caps, dtype=np.int64)
    h = C.c_void_p()
    _check(ctx, LIB.ns_featurize_tables(ctx, _ptr(desc), offsets.ctypes.data, caps.ctypes.data,
                                        len(caps), C.byref(h)))
    T_max = int(np.max(np.diff(offsets)))
    return Tables(ctx, h.value, offsets, T_max)


def ns_tables_single_costs(ctx: int, tables: Tables, features: bool = False):
    n = int(tables.offsets[-1])
    c = np.zeros(n)
    f = np.zeros((n, 5)) if features else None
    _check(ctx, LIB.ns_tables_single_costs(ctx, tables.handle, c.ctypes.data, _ptr(f)))
    return (c, f) if features else c


# ----------------------------------------------------------------- scoring
def ns_score_plans(ctx: int, tables: Tables, task: int, D: int, col_plan, assign, mode: int = NS_SCORE_FP64,
                   cost_out=None):
    """assign: int8 [P, T + n_col] numpy or CUDA tensor.  Returns
    (cost_out, best_index, best_cost); cost_out is a new host array unless
    one (host array or CUDA tensor) is given."""
    col = np.ascontiguousarray(col_plan if col_plan is not None else [], dtype=np.int32)
    P = int(assign.shape[0])
    if cost_out is None:
        cost_out = np.zeros(P)
    bi, bc = C.c_int64(), C.c_double()
    _check(ctx, LIB.ns_score_plans(ctx, tables.handle, task, D, col.ctypes.data if len(col) else None, len(col),
                                   _ptr(assign), P, mode, _ptr(cost_out), C.byref(bi), C.byref(bc)))
    return cost_out, bi.value, bc.value


# ----------------------------------------------------------------- search
NS_GREEDY_AUTO, NS_GREEDY_GROUPED, NS_GREEDY_LANES = 0, 1, 2
NS_SEARCH_ASYNC = 4


NS_NO_DIM_CAP = 8
NS_R10_ABS_STARTS, NS_R11_SUM_OF_MAX, NS_R14_SPLITTABLE = 16, 32, 64   # alternative readings


def _params(N, K, L, M, hi, greedy=NS_GREEDY_AUTO, async_=False, no_dim_cap=False, readings=0):
    return ns_search_params(N, K, L, M, hi, greedy | (NS_SEARCH_ASYNC if async_ else 0) |
                            (NS_NO_DIM_CAP if no_dim_cap else 0) | readings)


def _alloc_out(n: int, stride: int, L: int, out: Optional[dict]):
    if out is None:
        out = dict(cost=np.zeros(n), n_col=np.zeros(n, np.int32), col_plan=np.zeros((n, max(L, 1)), np.int32),
                   assign=np.zeros((n, stride), np.int8), grid_index=np.zeros(n, np.int32),
                   n_scores=np.zeros(n, np.uint64))
    pb = ns_plan_batch(_ptr(out["cost"]), _ptr(out.get("n_col")), _ptr(out.get("col_plan")),
                       _ptr(out.get("assign")), int(out["assign"].shape[1]) if out.get("assign") is not None else 0,
                       _ptr(out.get("grid_index")), _ptr(out.get("n_scores")))
    return out, pb


def ns_shard_tablewise(ctx: int, tables: Tables, D: int, M: int = 11, hi: float = 1.5, out: Optional[dict] = None,
                       greedy: int = NS_GREEDY_AUTO, async_: bool = False, no_dim_cap: bool = False,
                       readings: int = 0):
    """async_=True: NS_SEARCH_ASYNC (returns after enqueueing; sync before reading out);
    no_dim_cap=True: NS_NO_DIM_CAP (Table 3 "w/o greedy grid search", M must be 1)."""
    out, pb = _alloc_out(tables.n_tasks, tables.T_max, 0, out)
    p = _params(10, 3, 0, M, hi, greedy, async_, no_dim_cap, readings)
    st = _check(ctx, LIB.ns_shard_tablewise(ctx, tables.handle, D, C.byref(p), C.byref(pb)))
    out["status"] = st
    return out


def ns_shard_columnwise(ctx: int, tables: Tables, D: int, N: int = 10, K: int = 3, L: int = 10, M: int = 11,
                        hi: float = 1.5, out: Optional[dict] = None, greedy: int = NS_GREEDY_AUTO,
                        async_: bool = False, no_dim_cap: bool = False, readings: int = 0):
    out, pb = _alloc_out(tables.n_tasks, tables.T_max + L, L, out)
    p = _params(N, K, L, M, hi, greedy, async_, no_dim_cap, readings)
    st = _check(ctx, LIB.ns_shard_columnwise(ctx, tables.handle, D, C.byref(p), C.byref(pb)))
    out["status"] = st
    return out


# ----------------------------------------------------------------- workspace
_WORKSPACES = {}   # ctx -> the caller's tensor (kept alive while the ctx may use it)


def ns_set_workspace(ctx: int, buf) -> None:
    """Caller-owned device scratch (header: ns_set_workspace): ``buf`` is a
    CUDA tensor (e.g. torch.empty(n, dtype=torch.uint8, device="cuda")) or None
    to return to the library's own arena.  Marshalling only."""
    if buf is None:
        _check(ctx, LIB.ns_set_workspace(ctx, None, 0))
        _WORKSPACES.pop(ctx, None)
        return
    _check(ctx, LIB.ns_set_workspace(ctx, _dp(buf), buf.numel() * buf.element_size()))
    _WORKSPACES[ctx] = buf


def ns_search_workspace_bytes(ctx: int, n_tasks: int, T_max: int, D: int, columnwise: bool, N: int = 10,
                              K: int = 3, L: int = 10, M: int = 11, hi: float = 1.5, greedy: int = NS_GREEDY_AUTO) -> int:
    n = C.c_size_t(0)
    p = _params(N, K, L if columnwise else 0, M, hi, greedy)
    _check(ctx, LIB.ns_search_workspace_bytes(ctx, n_tasks, T_max, D, C.byref(p), 1 if columnwise else 0,
                                              C.byref(n)))
    return int(n.value)


def ns_score_workspace_bytes(ctx: int, T_prime: int, D: int, P: int, assign_on_device: bool) -> int:
    n = C.c_size_t(0)
    _check(ctx, LIB.ns_score_workspace_bytes(ctx, T_prime, D, P, 1 if assign_on_device else 0, C.byref(n)))
    return int(n.value)


# ----------------------------------------------------------------- comm
def ns_comm_unique_id() -> bytes:
    buf = (C.c_ubyte * 128)()
    st = LIB.ns_comm_unique_id(buf)
    if st != 0:
        raise NSError(st, "ns_comm_unique_id")
    return bytes(buf)


def ns_comm_init(ctx: int, nranks: int, rank: int, uid: Optional[bytes]) -> None:
    """uid None with nranks > 1: emulated ranks (test hook, no NCCL)."""
    buf = (C.c_ubyte * 128).from_buffer_copy(uid) if uid else None
    _check(ctx, LIB.ns_comm_init(ctx, nranks, rank, buf))


NS_COMM_MIN_U64 = 0
NS_COMM_MAX_I8 = 1
_HOST_COMMS = {}   # ctx -> (struct, callbacks): kept alive while the ctx uses them


def ns_comm_init_host(ctx: int, nranks: int, rank: int, allgather, allreduce, alltoallv=None) -> None:
    """Collectives through Python callbacks on host buffers (header:
    ns_host_comm).  ``allgather(send: np.ndarray[uint8], recv: np.ndarray[uint8])``
    fills recv (nranks blocks); ``allreduce(buf: np.ndarray, op)`` reduces in
    place (uint64 min or int8 max); ``alltoallv(send, send_bytes, recv,
    recv_bytes)`` (uint8 arrays, per-peer byte counts; optional, needed by the
    embedding-bag exchange).  Marshalling only."""
    def _report():   # a failing callback is reported to the caller as NS_ERR_NCCL
        import traceback
        traceback.print_exc()
        return 1

    def ag(user, send, recv, nbytes):
        try:
            s_ = np.ctypeslib.as_array((C.c_uint8 * nbytes).from_address(send))
            r_ = np.ctypeslib.as_array((C.c_uint8 * (nbytes * nranks)).from_address(recv))
            allgather(s_.copy(), r_)
            return 0
        except BaseException:
            return _report()

    def ar(user, buf, count, op):
        try:
            ct = C.c_uint64 if op == NS_COMM_MIN_U64 else C.c_int8
            b_ = np.ctypeslib.as_array((ct * count).from_address(buf))
            allreduce(b_, op)
            return 0
        except BaseException:
            return _report()

    def a2a(user, send, send_bytes, recv, recv_bytes):
        try:
            sb = [int(send_bytes[q]) for q in range(nranks)]
            rb = [int(recv_bytes[q]) for q in range(nranks)]
            s_ = np.ctypeslib.as_array((C.c_uint8 * max(sum(sb), 1)).from_address(send))[:sum(sb)]
            r_ = np.ctypeslib.as_array((C.c_uint8 * max(sum(rb), 1)).from_address(recv))[:sum(rb)]
            alltoallv(s_.copy(), sb, r_, rb)
            return 0
        except BaseException:
            return _report()

    cb = ns_host_comm(None, _ALLGATHER_FN(ag), _ALLREDUCE_FN(ar),
                      _ALLTOALLV_FN(a2a) if alltoallv is not None else _ALLTOALLV_FN())
    _HOST_COMMS[ctx] = cb
    _check(ctx, LIB.ns_comm_init_host(ctx, nranks, rank, C.byref(cb)))


def torch_host_alltoallv(group=None):
    """alltoallv callback over a torch.distributed process group (gloo:
    point-to-point send/recv of each peer's block, the self block copied)."""
    import torch
    import torch.distributed as dist

    def alltoallv(send, send_bytes, recv, recv_bytes):
        me = dist.get_rank(group)
        so = np.concatenate([[0], np.cumsum(send_bytes)]).astype(np.int64)
        ro = np.concatenate([[0], np.cumsum(recv_bytes)]).astype(np.int64)
        reqs = []
        for q in range(len(send_bytes)):
            if q == me:
                recv[ro[q]:ro[q + 1]] = send[so[q]:so[q + 1]]
                continue
            if send_bytes[q]:
                reqs.append(dist.isend(torch.from_numpy(send[so[q]:so[q + 1]].copy()), q, group=group))
        bufs = {}
        for r in range(len(recv_bytes)):
            if r != me and recv_bytes[r]:
                bufs[r] = torch.empty(int(recv_bytes[r]), dtype=torch.uint8)
                reqs.append(dist.irecv(bufs[r], r, group=group))
        for rq in reqs:
            rq.wait()
        for r, t in bufs.items():
            recv[ro[r]:ro[r + 1]] = t.numpy()

    return alltoallv


def torch_host_comm(group=None):
    """(allgather, allreduce) callbacks over a torch.distributed process group
    (e.g. gloo) for ns_comm_init_host."""
    import torch
    import torch.distributed as dist

    def allgather(send, recv):
        world = dist.get_world_size(group)
        t = torch.from_numpy(send)
        outs = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(outs, t, group=group)
        recv[:] = torch.cat(outs).numpy()

    def allreduce(buf, op):
        if op == NS_COMM_MIN_U64:
            # uint64 order == int64 order after flipping the sign bit
            v = torch.from_numpy(buf.view(np.int64) ^ np.int64(-0x8000000000000000))
            dist.all_reduce(v, op=dist.ReduceOp.MIN, group=group)
            buf[:] = (v.numpy() ^ np.int64(-0x8000000000000000)).view(np.uint64)
        else:
            v = torch.from_numpy(buf.astype(np.int32))   # int8 max via int32 (gloo-safe)
            dist.all_reduce(v, op=dist.ReduceOp.MAX, group=group)
            buf[:] = v.numpy().astype(np.int8)

    return allgather, allreduce


# ----------------------------------------------------------------- pre-training (F2)
def _dp(t):
    """Device pointer of a CUDA torch tensor (marshalling only)."""
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("pre-training buffers must be CUDA tensors")
    return t.data_ptr()


def ns_pretrain_compute_samples(ctx: int, pool_desc, aug_dims, comb_off, comb_idx, feats_out, labels_out) -> None:
    """Alg. 4 samples: features [rows][5] and labels [n] (device tensors)."""
    n_pool = pool_desc.numel() // TABLE_DESC.itemsize
    _check(ctx, LIB.ns_pretrain_compute_samples(ctx, _dp(pool_desc), n_pool, _dp(aug_dims), aug_dims.numel(),
                                                _dp(comb_off), _dp(comb_idx), comb_off.numel() - 1, _dp(feats_out),
                                                _dp(labels_out)))


def ns_pretrain_comm_samples(ctx: int, pool_desc, aug_dims, D: int, mem_cap: int, off, idx, p, u, r, starts,
                             x_out, yf_out, yb_out, assign_out, valid_out) -> None:
    """Alg. 5 placements and their comm labels (device tensors)."""
    n_pool = pool_desc.numel() // TABLE_DESC.itemsize
    _check(ctx, LIB.ns_pretrain_comm_samples(ctx, _dp(pool_desc), n_pool, _dp(aug_dims), aug_dims.numel(), D, mem_cap,
                                             _dp(off), _dp(idx), _dp(p), _dp(u), _dp(r), _dp(starts), off.numel() - 1,
                                             _dp(x_out), _dp(yf_out), _dp(yb_out), _dp(assign_out), _dp(valid_out)))


def ns_pretrain_compute_step(ctx: int, theta, m, v, t: int, lr: float, feats, off, labels, batch, max_rows: int,
                             loss_out=None) -> None:
    _check(ctx, LIB.ns_pretrain_compute_step(ctx, _dp(theta), _dp(m), _dp(v), t, lr, _dp(feats), _dp(off),
                                             _dp(labels), _dp(batch), batch.numel(), max_rows, _dp(loss_out)))


def ns_pretrain_comm_step(ctx: int, D: int, theta, m, v, t: int, lr: float, x, y, batch, loss_out=None) -> None:
    _check(ctx, LIB.ns_pretrain_comm_step(ctx, D, _dp(theta), _dp(m), _dp(v), t, lr, _dp(x), _dp(y), _dp(batch),
                                          batch.numel(), _dp(loss_out)))


# ----------------------------------------------------------------- real-cost evaluator (F3)
def _bag_tables(tables):
    """tables: sequence of (weights [rows][dim] f32, indices i64, offsets i32) CUDA tensors."""
    arr = (ns_bag_table * len(tables))()
    for k, (W, idx, off) in enumerate(tables):
        arr[k] = ns_bag_table(int(W.shape[1]), 0, int(W.shape[0]), _dp(W), _dp(idx) if idx.numel() else None,
                              _dp(off))
    return arr


def ns_embedding_bag_forward(ctx: int, tables, batch: int, out) -> None:
    arr = _bag_tables(tables)
    _check(ctx, LIB.ns_embedding_bag_forward(ctx, arr, len(tables), batch, _dp(out)))


def ns_embedding_bag_backward_sgd(ctx: int, tables, batch: int, grad_out, lr: float) -> None:
    arr = _bag_tables(tables)
    _check(ctx, LIB.ns_embedding_bag_backward_sgd(ctx, arr, len(tables), batch, _dp(grad_out), lr))


def _cols_arg(cols):
    a = (C.c_int32 * len(cols))(*[int(c) for c in cols])
    return a


def ns_embedding_bag_forward_exchange(ctx: int, tables, batch: int, cols, out, recv) -> None:
    """Forward + all-to-all (header: ns_embedding_bag_forward_exchange); cols
    = per-rank sums of table dims (host list)."""
    arr = _bag_tables(tables)
    _check(ctx, LIB.ns_embedding_bag_forward_exchange(ctx, arr, len(tables), batch, _cols_arg(cols), _dp(out),
                                                      _dp(recv)))


def ns_embedding_bag_backward_exchange_sgd(ctx: int, tables, batch: int, cols, grad_recv, grad_out,
                                           lr: float) -> None:
    arr = _bag_tables(tables)
    _check(ctx, LIB.ns_embedding_bag_backward_exchange_sgd(ctx, arr, len(tables), batch, _cols_arg(cols),
                                                           _dp(grad_recv), _dp(grad_out), lr))
