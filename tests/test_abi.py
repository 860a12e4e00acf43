"""CPU checks of the C-ABI library: it loads, exports every symbol that
include/neuroshard.h declares, the ctypes structures match the header's
layout, and argument validation works without a GPU."""
import ctypes as C
import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "neuroshard.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ns_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    import paper_2305_01868_b200 as ns
    lib = C.CDLL(ns.LIB_PATH)
    names = _declared()
    assert {"ns_load_cost_models", "ns_featurize_tables", "ns_score_plans", "ns_shard_tablewise",
            "ns_shard_columnwise"} <= set(names)
    for n in names:
        assert hasattr(lib, n), f"{n} declared in neuroshard.h but not exported"
    assert set(ns.EXPORTED) == set(names)


def test_struct_layouts():
    from paper_2305_01868_b200 import _native as nv
    assert C.sizeof(nv.ns_linear) == 24
    assert C.sizeof(nv.ns_compute_model) == 4 * 24
    assert C.sizeof(nv.ns_comm_model) == 8 + 5 * 24 + 16
    assert C.sizeof(nv.ns_search_params) == 32
    assert C.sizeof(nv.ns_plan_batch) == 7 * 8
    assert nv.TABLE_DESC.itemsize == 32


def test_no_gpu_is_an_error_not_a_fallback():
    import torch
    from paper_2305_01868_b200 import _native as nv
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = C.c_void_p()
    st = nv.LIB.ns_create(C.byref(h), 0, None)
    assert st == -4 and not h.value   # NS_ERR_CUDA


def test_null_arguments_rejected():
    from paper_2305_01868_b200 import _native as nv
    assert nv.LIB.ns_create(None, 0, None) == -1
    assert nv.LIB.ns_destroy(None) == -1
    assert nv.LIB.ns_shard_tablewise(None, None, 4, None, None) == -1
    assert nv.LIB.ns_score_plans(None, None, 0, 4, None, 0, None, 1, 0, None, None, None) == -1
    assert nv.LIB.ns_comm_unique_id(None) == -1


def test_oracle_and_product_are_independent():
    """The product package must not import the oracle and vice versa."""
    pkg = os.path.join(ROOT, "paper_2305_01868_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\w+)", txt, re.M), f
    for f in os.listdir(os.path.join(ROOT, "oracle")):
        if f.endswith(".py"):
            txt = open(os.path.join(ROOT, "oracle", f)).read()
            assert "paper_2305_01868_b200" not in re.findall(r"^\s*(?:from|import)\s+(\w+)", txt, re.M), f


def test_batching_service_without_gpu_raises():
    """The batching service's worker reports the ctx failure to the caller
    (no silent CPU path)."""
    import torch
    from paper_2305_01868_b200 import NSError, ShardingService
    from workload.synth import gen_weights
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(NSError):
        ShardingService(gen_weights(4, "mono"), 4)
