"""f2: the minimax (bottleneck) path algebra (§6) through
every call of the C ABI, vs the oracle's minimax FW (bit-exact: max and min
are exact in int32 and fp32, so fp32 is compared exactly too)."""
import dataclasses

import numpy as np
import pytest

import oracle
import synth
from conftest import random_graph

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

INF = synth.INF_I32


@pytest.fixture(scope="module")
def lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2412_15122_b200 as P
    return P


def make(P, W, directed=True, cap=None):
    return P.WarmAPSP(torch.from_numpy(np.ascontiguousarray(W)), directed=directed, cap=cap,
                      semiring="minimax")


def getD(h):
    torch.cuda.synchronize()
    return h.D.cpu().numpy()


def exact(G, O):
    G, O = np.asarray(G), np.asarray(O)
    if np.issubdtype(G.dtype, np.floating):
        O = O.astype(np.float32)
    bad = np.argwhere(G != O)
    assert bad.size == 0, f"{len(bad)} mismatches, first {bad[:3].tolist()}"


@pytest.mark.parametrize("n", [2, 129, 300])
@pytest.mark.parametrize("directed", [True, False])
def test_minimax_cold_fw(lib, rng, n, directed):
    W = random_graph(rng, n, directed, 0.5, lo=0, hi=1000, inf_frac=0.05)
    exact(getD(make(lib, W, directed)), oracle.fw_minimax(W))


def test_minimax_cold_fw_fp32(lib):
    spec = dataclasses.replace(synth.C2, n=260)
    W = synth.graph(spec)
    exact(getD(make(lib, W, False)), oracle.fw_minimax(W))


@pytest.mark.parametrize("directed", [True, False])
def test_minimax_sequence(lib, rng, directed):
    """Adds, removals, decreases and increases (random and tight) in the
    minimax algebra; both recompute paths."""
    n = 180
    W = random_graph(rng, n, directed, 0.8, lo=1, hi=500)
    cap = n + 8
    h = make(lib, W, directed, cap)
    hg = synth.HostGraph(W, directed, cap=cap)
    for t in range(14):
        kind = t % 4
        if kind == 0:
            o = rng.integers(1, 500, hg.n).astype(np.int32)
            i = o.copy() if not directed else rng.integers(1, 500, hg.n).astype(np.int32)
            h.add_node(o, i)
            hg.add_node(o, i)
        elif kind == 1:
            h.set_option(0, (t // 4) % 3)
            k = int(rng.integers(hg.n))
            h.remove_node(k)
            hg.remove_node(k)
        else:
            u, v = (int(x) for x in rng.choice(hg.n, 2, replace=False))
            D = getD(h)
            if kind == 2:
                w = max(0, int(D[u, v]) - 1)          # below the bottleneck: changes entries
            else:
                row = hg.W[u].astype(np.int64)
                row[u] = 1 << 40
                v = int(np.argmin(row))
                w = int(hg.weight(u, v)) * 3 + 1      # raise the cheapest edge (tight)
            h.update_edge(u, v, w)
            hg.set_edge(u, v, w)
        exact(getD(h), oracle.fw_minimax(hg.W))


def test_minimax_modify_readd(lib, rng):
    n = 120
    W = random_graph(rng, n, True, 1.0, lo=1, hi=300)
    h = make(lib, W)
    for trial in range(4):
        u, v = (int(x) for x in rng.choice(n, 2, replace=False))
        w = int(rng.integers(1, 600))
        h.modify_edge_readd(u, v, w)
        W[u, v] = w
        exact(getD(h), oracle.fw_minimax(W))


def test_minimax_queries(lib, rng):
    """alg:sp_apsp in the minimax algebra: the path's largest edge equals D[s][t]."""
    n = 200
    W = random_graph(rng, n, True, 0.4, lo=1, hi=1000)
    h = make(lib, W)
    D = getD(h)
    for _ in range(30):
        s, t = (int(x) for x in rng.integers(0, n, 2))
        d, path, nc = h.query(s, t, path_cap=n)
        assert d == D[s, t]
        if s == t:
            assert path == [s]
        elif D[s, t] == INF:
            assert path == []
        else:
            assert oracle.path_is_valid(W, path, s, t)
            assert max(int(W[a, b]) for a, b in zip(path[:-1], path[1:])) == d
