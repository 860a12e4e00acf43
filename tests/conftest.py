import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from workload.synth import Task, Weights  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu)")
    config.addinivalue_line("markers", "slow: slower CPU test")


def load_golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def _sparse(shape, entries):
    a = np.zeros(shape)
    for e in entries:
        if len(shape) == 2:
            a[e[0], e[1]] = e[2]
        else:
            a[e[0]] = e[1]
    return a


def hand_weights(g):
    """Build the hand-example weights of tests/golden/hand_example.json."""
    w = g["weights"]
    D = g["D"]
    enc = [(_sparse((128, 5), w["enc1"]), np.zeros(128)),
           (_sparse((32, 128), w["enc2"]), np.zeros(32))]
    head = [(_sparse((64, 32), w["head1"]), _sparse((64,), w["head1_bias"])),
            (_sparse((1, 64), w["head2"]), _sparse((1,), w["head2_bias"]))]
    widths = [2 * D, 128, 64, 32, 16, D]
    n = w["comm_identity_units"]

    def comm(last, last_b):
        layers = []
        for j in range(4):
            W = np.zeros((widths[j + 1], widths[j]))
            for i in range(n):
                W[i, i] = 1.0
            layers.append((W, np.zeros(widths[j + 1])))
        layers.append((_sparse((D, 16), last), _sparse((D,), last_b)))
        return layers

    return Weights(enc=enc, head=head, comm_fwd=comm(w["fwd5"], w["fwd5_bias"]),
                   comm_bwd=comm(w["bwd5"], w["bwd5_bias"]), D=D, kind="hand")


def hand_task(g):
    t = g["tables"]
    return Task(np.array(t["dims"], np.int32), np.array(t["hash"], np.int64),
                np.array(t["pooling"], np.float64), np.array(t["skew"], np.float64),
                g["D"], int(g["cap"]), seed=0)


def small_task(rng, T, D, cap=4 << 30, max_dim=128, hash_hi=1e6):
    dims = (4 * rng.integers(1, max_dim // 4 + 1, size=T)).astype(np.int32)
    hash_ = np.rint(np.exp(rng.uniform(np.log(1e4), np.log(hash_hi), size=T))).astype(np.int64)
    pooling = np.exp(rng.uniform(0.0, np.log(60.0), size=T))
    skew = rng.uniform(0.0, 2.0, size=T)
    return Task(dims, hash_, pooling, skew, D, int(cap), seed=-1)


@pytest.fixture
def golden_hand():
    return load_golden("hand_example.json")
