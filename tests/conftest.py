import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


def load_golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def golden_graph(g, dtype=np.int32):
    """Dense W (diag 0, absent INF) from a golden fixture's edge list."""
    import synth

    names = g["nodes"]
    idx = {a: i for i, a in enumerate(names)}
    n = len(names)
    inf = synth.INF_I32 if dtype == np.int32 else np.inf
    W = np.full((n, n), inf, dtype=dtype)
    np.fill_diagonal(W, 0)
    for a, b, w in g["edges"]:
        W[idx[a], idx[b]] = w
        if not g["directed"]:
            W[idx[b], idx[a]] = w
    return W, idx


def random_graph(rng, n, directed=True, density=1.0, lo=0, hi=5, dtype=np.int32, inf_frac=0.0):
    """Small random test graph (tests only): integer weights in [lo, hi]."""
    import synth

    inf = synth.INF_I32 if dtype == np.int32 else np.float32(np.inf)
    if dtype == np.int32:
        W = rng.integers(lo, hi + 1, size=(n, n)).astype(np.int32)
    else:
        W = (rng.integers(1, 1 << 24, size=(n, n)).astype(np.float64) * 2.0 ** -24 * hi).astype(np.float32)
    present = rng.random((n, n)) < density
    if inf_frac:
        present &= rng.random((n, n)) >= inf_frac
    W = np.where(present, W, inf).astype(dtype)
    if not directed:
        W = np.triu(W, 1)
        W = W + W.T
        if dtype == np.int32:
            # re-apply INF symmetrically (the sum above doubled INF entries)
            up = np.triu(present, 1)
            mask = up | up.T
            W = np.where(mask, W, inf).astype(dtype)
    np.fill_diagonal(W, 0)
    return W


@pytest.fixture
def rng():
    return np.random.default_rng(12345)
