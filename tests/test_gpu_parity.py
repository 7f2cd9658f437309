"""GPU parity: every hot-path call through the C ABI vs the CPU oracle.

int32: bit-exact.  fp32: |g - o| <= 1e-5 |o| per entry, with 0 and inf
matching exactly (BASELINE.json north_star).
"""
import dataclasses

import numpy as np
import pytest

import oracle
import synth
from conftest import golden_graph, load_golden, random_graph

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

INF = synth.INF_I32
RTOL = 1e-5


@pytest.fixture(scope="module")
def lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2412_15122_b200 as P
    return P


def make(P, W, directed=True, cap=None, cold=True):
    return P.WarmAPSP(torch.from_numpy(np.ascontiguousarray(W)), directed=directed, cap=cap,
                      cold_start=cold)


def getD(h):
    torch.cuda.synchronize()
    return h.D.cpu().numpy()


def assert_parity(G, O):
    G = np.asarray(G)
    O = np.asarray(O)
    assert G.shape == O.shape
    if np.issubdtype(G.dtype, np.integer):
        bad = np.argwhere(G != O)
        assert bad.size == 0, f"{len(bad)} mismatches, first {bad[:5].tolist()}: gpu {G[tuple(bad[0])]} oracle {O[tuple(bad[0])]}"
    else:
        Gd = G.astype(np.float64)
        fin = np.isfinite(O)
        assert np.array_equal(np.isfinite(Gd), fin), "inf pattern differs"
        assert np.array_equal(Gd[O == 0] == 0, np.ones(np.count_nonzero(O == 0), bool)), "zeros differ"
        rel = np.abs(Gd[fin] - O[fin]) / np.maximum(np.abs(O[fin]), 1e-300)
        assert rel.max(initial=0) <= RTOL, f"max rel err {rel.max()}"


# ------------------------------------------------------------------ cold FW (a1)
@pytest.mark.parametrize("n", [1, 2, 5, 127, 128, 129, 255, 300, 513])
@pytest.mark.parametrize("directed", [True, False])
def test_cold_fw_int32(lib, rng, n, directed):
    W = random_graph(rng, n, directed, density=0.5, lo=0, hi=40, inf_frac=0.1)
    h = make(lib, W, directed)
    assert_parity(getD(h), oracle.fw(W))


def test_cold_fw_int32_bj_c1(lib):
    W = synth.graph(synth.C1)
    h = make(lib, W)
    assert_parity(getD(h), oracle.fw(W))


@pytest.mark.parametrize("n", [3, 130, 400])
def test_cold_fw_fp32(lib, n):
    spec = dataclasses.replace(synth.C2, n=n)
    W = synth.graph(spec)
    h = make(lib, W, directed=False)
    G = getD(h)
    assert_parity(G, oracle.fw(W))
    assert np.array_equal(G, G.T)   # Q17: FW keeps exact symmetry


def test_cold_fw_closed_form_cycle(lib):
    n = 1500
    W = np.full((n, n), INF, np.int32)
    np.fill_diagonal(W, 0)
    W[np.arange(n), (np.arange(n) + 1) % n] = 1
    h = make(lib, W)
    i, j = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    assert_parity(getD(h), ((j - i) % n).astype(np.int32))


def test_cold_fw_disconnected(lib, rng):
    W = random_graph(rng, 200, True, density=0.02, lo=1, hi=9)
    h = make(lib, W)
    assert_parity(getD(h), oracle.fw(W))


# ------------------------------------------------------------------ add node (a2)
def test_add_node_bj_c1(lib):
    """BJ.c1: n=256, add one node with U[1,100] edges; warm == cold FW."""
    spec = synth.C1
    W = synth.graph(spec)
    hg = synth.HostGraph(W, True, cap=257)
    o, i = synth.node_edges(spec, 0, 256)
    h = make(lib, W, cap=257)
    x, info = h.add_node(o, i)
    assert x == 256 and info.kind == 3 and h.n == 257
    hg.add_node(o, i)
    assert_parity(getD(h), oracle.fw(hg.W))


@pytest.mark.parametrize("directed", [True, False])
@pytest.mark.parametrize("n", [1, 7, 129, 1030])
def test_add_node_random(lib, rng, n, directed):
    W = random_graph(rng, n, directed, density=0.6, lo=0, hi=30, inf_frac=0.05)
    o = rng.integers(0, 30, n).astype(np.int32)
    o[rng.random(n) < 0.2] = INF
    i = o.copy() if not directed else rng.integers(0, 30, n).astype(np.int32)
    h = make(lib, W, directed, cap=n + 3)
    h.add_node(o, i)
    hg = synth.HostGraph(W, directed, cap=n + 3)
    hg.add_node(o, i)
    assert_parity(getD(h), oracle.fw(hg.W))


def test_add_node_golden_one_node(lib):
    g = load_golden("add_one_node.json")
    h = make(lib, np.zeros((1, 1), np.int32), cap=2)
    h.add_node(np.array(g["out_w"], np.int32), np.array(g["in_w"], np.int32))
    assert getD(h).tolist() == g["expected"]


def test_add_isolated_node_is_noop(lib, rng):
    W = random_graph(rng, 100, True, 1.0, lo=1, hi=50)
    h = make(lib, W, cap=101)
    D0 = getD(h).copy()
    h.add_node(np.full(100, INF, np.int32), np.full(100, INF, np.int32))
    D = getD(h)
    assert np.array_equal(D[:100, :100], D0)
    assert np.all(D[100, :100] == INF) and np.all(D[:100, 100] == INF) and D[100, 100] == 0


def test_add_hub_changes_every_entry(lib):
    """Closed form: hub with edges c/4 on a complete graph of
    uniform weight c -> every old off-diagonal distance becomes c/2."""
    n, c = 300, 40
    W = np.full((n, n), c, np.int32)
    np.fill_diagonal(W, 0)
    h = make(lib, W, cap=n + 1)
    h.add_node(np.full(n, c // 4, np.int32), np.full(n, c // 4, np.int32))
    D = getD(h)
    exp = np.full((n + 1, n + 1), c // 2, np.int32)
    exp[n, :] = c // 4
    exp[:, n] = c // 4
    np.fill_diagonal(exp, 0)
    assert_parity(D, exp)


def test_add_node_fp32_undirected(lib):
    spec = dataclasses.replace(synth.C2, n=300)
    W = synth.graph(spec)
    o, i = synth.node_edges(spec, 5, 300)
    h = make(lib, W, directed=False, cap=301)
    h.add_node(o, i)
    hg = synth.HostGraph(W, False, cap=301)
    hg.add_node(o, i)
    assert_parity(getD(h), oracle.fw(hg.W))


def test_recursion_cold_start_by_adds(lib, rng):
    """Algorithm 1 idea: n successive add-nodes from one node == cold FW."""
    n = 60
    W = random_graph(rng, n, True, 0.7, lo=1, hi=20)
    h = make(lib, W[:1, :1], cap=n)
    for x in range(1, n):
        h.add_node(W[x, :x].copy(), W[:x, x].copy())
    assert_parity(getD(h), oracle.fw(W))


# ------------------------------------------------------------------ edge updates (a3, a4)
def _edit(W, u, v, w, directed):
    W2 = W.copy()
    W2[u, v] = w
    if not directed:
        W2[v, u] = w
    return W2


@pytest.mark.parametrize("directed", [True, False])
def test_decrease_random_and_tight(lib, rng, directed):
    n = 260
    W = random_graph(rng, n, directed, 1.0, lo=1, hi=100)
    h = make(lib, W, directed)
    for trial in range(12):
        D = getD(h)
        u, v = (int(x) for x in rng.choice(n, 2, replace=False))
        w_old = int(W[u, v])
        if trial % 2:
            w_new = max(0, int(D[u, v]) // 2)    # tight variant: always changes entries
        else:
            w_new = max(0, w_old // 10)
        if w_new >= w_old:
            continue
        info = h.update_edge(u, v, w_new)
        W = _edit(W, u, v, w_new, directed)
        assert info.kind == 1
        assert info.early_exit == (w_new >= D[u, v])
        assert_parity(getD(h), oracle.fw(W))


def test_decrease_closed_form_chord(lib):
    n = 700
    W = np.full((n, n), INF, np.int32)
    np.fill_diagonal(W, 0)
    W[np.arange(n), (np.arange(n) + 1) % n] = 1
    h = make(lib, W)
    u, v = 10, 400
    h.update_edge(u, v, 1)
    i, j = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    exp = np.minimum((j - i) % n, (u - i) % n + 1 + (j - v) % n)
    assert_parity(getD(h), exp.astype(np.int32))


@pytest.mark.parametrize("directed", [True, False])
@pytest.mark.parametrize("force", [0, 1, 2])
def test_increase_random_and_tight(lib, rng, directed, force):
    n = 230
    W = random_graph(rng, n, directed, 1.0, lo=1, hi=60)
    h = make(lib, W, directed)
    h.set_option(0, force)
    for trial in range(8):
        D = getD(h)
        if trial % 2:
            u = int(rng.integers(n))
            row = W[u].astype(np.int64)
            row[u] = np.iinfo(np.int64).max
            v = int(np.argmin(row))            # cheapest out-edge: always tight
        else:
            u, v = (int(x) for x in rng.choice(n, 2, replace=False))
        w_old = int(W[u, v])
        w_new = int(rng.choice([w_old * 10, w_old + 1, INF]))
        info = h.update_edge(u, v, w_new)
        tight = w_old == D[u, v]
        mask = oracle.need_update_increase(D, u, v, w_old, directed)
        W = _edit(W, u, v, w_new, directed)
        assert info.kind == 2 and info.early_exit == (not tight)
        if tight:
            assert info.affected_pairs == mask.sum()
            assert info.affected_rows == mask.any(axis=1).sum()
            assert info.path == (3 if force == 2 else 2) or (force == 0 and info.path in (2, 3))
        assert_parity(getD(h), oracle.fw(W))


def test_increase_closed_form_cycle_cut(lib):
    """Cycle edge u->u+1 set to INF: pairs whose arc crosses it become INF
    (|A| = Theta(n^2), forces the dense fallback by the gate)."""
    n = 400
    W = np.full((n, n), INF, np.int32)
    np.fill_diagonal(W, 0)
    W[np.arange(n), (np.arange(n) + 1) % n] = 1
    h = make(lib, W)
    u = 123
    info = h.update_edge(u, u + 1, INF)
    W2 = _edit(W, u, u + 1, INF, True)
    assert info.path == 3
    assert_parity(getD(h), oracle.fw(W2))


@pytest.mark.parametrize("force", [1, 2])
def test_edge_updates_fp32_undirected(lib, rng, force):
    spec = dataclasses.replace(synth.C2, n=320)
    W = synth.graph(spec)
    h = make(lib, W, directed=False)
    h.set_option(0, force)
    for trial in range(6):
        D = getD(h)
        u = int(rng.integers(320))
        if trial % 2 == 0:
            v = int(np.argmin(np.where(np.arange(320) == u, np.inf, W[u])))
            w_new = np.float32(W[u, v] * np.float32(10))     # tight increase
        else:
            v = int((u + 1 + rng.integers(319)) % 320)
            w_new = np.float32(D[u, v] * np.float32(0.5))    # tight decrease
        h.update_edge(u, v, float(w_new))
        W = _edit(W, u, v, w_new, False)
        assert_parity(getD(h), oracle.fw(W))


def test_insert_and_delete_edge(lib, rng):
    W = random_graph(rng, 150, True, 0.1, lo=1, hi=9)
    h = make(lib, W)
    absent = np.argwhere((W == INF))
    u, v = (int(x) for x in absent[len(absent) // 2])
    h.update_edge(u, v, 3)          # insert (decrease from INF)
    W = _edit(W, u, v, 3, True)
    assert_parity(getD(h), oracle.fw(W))
    h.update_edge(u, v, INF)        # delete (increase to INF)
    W = _edit(W, u, v, INF, True)
    assert_parity(getD(h), oracle.fw(W))


def test_decrease_then_restore_round_trip(lib, rng):
    W = random_graph(rng, 200, True, 1.0, lo=1, hi=100)
    h = make(lib, W)
    D0 = getD(h).copy()
    u, v = 3, 77
    h.update_edge(u, v, max(0, int(D0[u, v]) // 3))
    h.update_edge(u, v, int(W[u, v]))
    assert_parity(getD(h), D0)


# ------------------------------------------------------------------ remove node (a5-a7)
@pytest.mark.parametrize("directed", [True, False])
@pytest.mark.parametrize("force", [0, 1, 2])
def test_remove_random(lib, rng, directed, force):
    n = 260
    W = random_graph(rng, n, directed, 0.9, lo=1, hi=1000)
    h = make(lib, W, directed)
    h.set_option(0, force)
    hg = synth.HostGraph(W, directed)
    for trial in range(6):
        D = getD(h)
        k = int(rng.integers(hg.n))
        mask = oracle.need_update_removal(D, k)
        mf, info = h.remove_node(k)
        assert mf == (hg.n - 1 if k != hg.n - 1 else -1)
        hg.remove_node(k)
        assert info.kind == 4
        assert info.affected_pairs == mask.sum()
        phi, cost = oracle.cost(mask, D.shape[0])
        assert info.affected_rows == phi and abs(info.cost - cost) < 1e-12
        assert_parity(getD(h), oracle.fw(hg.W))


def test_remove_golden_hub(lib):
    g = load_golden("hub_remove.json")
    W, idx = golden_graph(g)
    h = make(lib, W, directed=False)
    mf, info = h.remove_node(idx["B"])
    assert info.affected_pairs == 4 and info.affected_rows == 3 and info.cost == g["cost"]
    hg = synth.HostGraph(W, False)
    hg.remove_node(idx["B"])
    assert_parity(getD(h), oracle.fw(hg.W))


def test_remove_golden_star_avoided(lib):
    g = load_golden("star_avoided_remove.json")
    W, idx = golden_graph(g)
    h = make(lib, W, directed=False)
    _, info = h.remove_node(idx["C"])
    assert info.affected_pairs == 0 and info.cost == 0.0


def test_remove_line_metric_ties_dense(lib):
    """Line metric: removing an interior point flags 2p(1-p)n^2 tie pairs but
    changes no value; exercises the gate and a7."""
    n = 301
    x = np.arange(n) * 3
    W = np.abs(x[:, None] - x[None, :]).astype(np.int32)
    h = make(lib, W)
    k = 150
    D = getD(h)
    mask = oracle.need_update_removal(D, k)
    _, info = h.remove_node(k)
    assert info.affected_pairs == mask.sum() > 0
    hg = synth.HostGraph(W, True)
    hg.remove_node(k)
    assert_parity(getD(h), oracle.fw(hg.W))


@pytest.mark.parametrize("force", [0, 1])
def test_list_overflow_recovers_through_dense(lib, force):
    """|A| ~ n^2/2 > the need_update_list capacity (max(cap^2/32, 2^20) pairs):
    the detection pass cannot list every pair, so the flagged entries are reset
    in place by a second pass (MODE 2) and blocked FW runs on D0 — also when
    the sparse path is forced.  Directed removal and undirected increase (the
    two-term detection)."""
    n = 2048
    x = np.arange(n) * 3
    W = np.abs(x[:, None] - x[None, :]).astype(np.int32)
    h = make(lib, W)
    h.set_option(0, force)
    _, info = h.remove_node(n // 2)
    assert info.affected_pairs > (1 << 20) and info.path == 3
    hg = synth.HostGraph(W, True)
    hg.remove_node(n // 2)
    assert_parity(getD(h), oracle.fw(hg.W))
    hu = make(lib, W, directed=False)
    hu.set_option(0, force)
    p = n // 2
    info = hu.update_edge(p, p + 1, 30)   # tight edge of the line: every crossing pair is flagged
    assert info.affected_pairs > (1 << 20) and info.path == 3
    assert_parity(getD(hu), oracle.fw(_edit(W, p, p + 1, 30, False)))


def test_remove_cycle_closed_form(lib):
    n = 500
    W = np.full((n, n), INF, np.int32)
    np.fill_diagonal(W, 0)
    W[np.arange(n), (np.arange(n) + 1) % n] = 1
    h = make(lib, W)
    k = n - 1   # no swap: pairs whose arc passes through k become INF
    h.remove_node(k)
    m = n - 1
    i, j = np.meshgrid(np.arange(m), np.arange(m), indexing="ij")
    exp = np.where(j >= i, j - i, INF).astype(np.int32)
    assert_parity(getD(h), exp)


def test_remove_then_readd_round_trip(lib, rng):
    W = random_graph(rng, 180, True, 1.0, lo=1, hi=100)
    h = make(lib, W)
    D0 = getD(h).copy()
    last = 179
    h.remove_node(last)
    h.add_node(W[last, :last].copy(), W[:last, last].copy())
    assert_parity(getD(h), D0)


@pytest.mark.parametrize("dtype", ["i32", "f32"])
def test_remove_fp32_and_density(lib, rng, dtype):
    if dtype == "i32":
        spec = dataclasses.replace(synth.C3, n=400)
    else:
        spec = dataclasses.replace(synth.C2, n=400)
    W = synth.graph(spec)
    h = make(lib, W, directed=spec.directed)
    hg = synth.HostGraph(W, spec.directed)
    for k in (0, 399 - 1, 200):
        h.remove_node(k)
        hg.remove_node(k)
        assert_parity(getD(h), oracle.fw(hg.W))


# ------------------------------------------------------------------ sequences (BJ.c4 shape)
def test_update_sequence_small(lib):
    spec = dataclasses.replace(synth.C4, n=384)
    W = synth.graph(spec)
    cap = 384 + 16
    hg = synth.HostGraph(W, True, cap=cap)
    h = make(lib, W, cap=cap)
    seq = synth.update_sequence(spec, synth.HostGraph(W, True, cap=cap), 0, 30)
    for up in seq:
        if up.kind == "add":
            h.add_node(up.out_w, up.in_w)
            hg.add_node(up.out_w, up.in_w)
        elif up.kind == "remove":
            h.remove_node(up.k)
            hg.remove_node(up.k)
        else:
            h.update_edge(up.u, up.v, up.w_new)
            hg.set_edge(up.u, up.v, up.w_new)
        assert h.n == hg.n
    assert_parity(getD(h), oracle.fw(hg.W))


# ------------------------------------------------------------------ query (a8)
def _check_path(W, D, s, t, dist, path):
    if s == t:
        assert path == [s] and dist == 0
        return
    if D[s, t] == INF or (np.issubdtype(np.asarray(D).dtype, np.floating) and not np.isfinite(D[s, t])):
        assert path == []
        return
    assert oracle.path_is_valid(W, path, s, t)
    pw = oracle.path_weight(W, path)
    if np.issubdtype(np.asarray(W).dtype, np.integer):
        assert pw == dist == D[s, t]
    else:
        assert abs(pw - dist) <= RTOL * abs(dist)
        assert abs(dist - D[s, t]) <= RTOL * abs(D[s, t])


def test_query_golden_hub(lib):
    g = load_golden("hub_query.json")
    W, idx = golden_graph(g)
    h = make(lib, W, directed=False)
    d, path, nc = h.query(idx["A"], idx["C"])
    assert d == g["dist"] and [g["nodes"][i] for i in path] == g["path"] and nc == 3


@pytest.mark.parametrize("directed", [True, False])
def test_query_random(lib, rng, directed):
    n = 300
    W = random_graph(rng, n, directed, 0.3, lo=1, hi=20, inf_frac=0.0)
    h = make(lib, W, directed)
    D = oracle.fw(W)                      # the oracle's matrix, not the GPU's
    for _ in range(40):
        s, t = (int(x) for x in rng.integers(0, n, 2))
        d, path, nc = h.query(s, t)
        dd, _ = oracle.dijkstra_pair(W, s, t)
        assert d == D[s, t] == (0 if s == t else dd)
        _check_path(W, D, s, t, d, path)
        if s != t and D[s, t] != INF:
            assert nc == len(oracle.candidates(D, s, t))


def test_query_zero_weights(lib, rng):
    n = 40
    W = random_graph(rng, n, True, 0.5, lo=0, hi=2)
    h = make(lib, W)
    D = oracle.fw(W)
    for s in range(0, n, 3):
        for t in range(1, n, 5):
            d, path, _ = h.query(s, t)
            _check_path(W, D, s, t, d, path)


def test_query_batch_matches_single(lib, rng):
    spec = dataclasses.replace(synth.C5, n=500)
    W = synth.graph(spec)
    h = make(lib, W)
    D = oracle.fw(W)
    s, t = synth.query_pairs(spec.seed, 500, 64)
    dist, paths, lens, nc = h.query_batch(s, t, path_cap=32)
    dist, paths, lens = dist.cpu().numpy(), paths.cpu().numpy(), lens.cpu().numpy()
    for q in range(64):
        assert dist[q] == D[s[q], t[q]]
        p = paths[q, : lens[q]].tolist()
        _check_path(W, D, int(s[q]), int(t[q]), dist[q], p)


def test_query_large_batch_grouped_by_t(lib, rng):
    """A batch beyond one launch pair (1024 queries) runs t-grouped (f3: the
    queries sorted by target, answers written back to their own slots):
    3000 queries over 40 targets, every answer vs the oracle's D and a valid
    shortest path; the same pairs one by one give the same paths' lengths."""
    spec = dataclasses.replace(synth.C5, n=400)
    W = synth.graph(spec)
    h = make(lib, W)
    D = oracle.fw(W)
    q = 3000
    s = rng.integers(0, 400, q).astype(np.int32)
    t = rng.choice(rng.permutation(400)[:40], q).astype(np.int32)
    dist, paths, lens, nc = h.query_batch(s, t, path_cap=64)
    dist, paths, lens, nc = dist.cpu().numpy(), paths.cpu().numpy(), lens.cpu().numpy(), nc.cpu().numpy()
    for k in range(q):
        assert dist[k] == D[s[k], t[k]], k
        p = paths[k, : lens[k]].tolist()
        _check_path(W, D, int(s[k]), int(t[k]), dist[k], p)
    for k in rng.choice(q, 20, replace=False):
        d1, p1, n1 = h.query(int(s[k]), int(t[k]), path_cap=64)
        assert d1 == dist[k] and len(p1) == lens[k] and n1 == nc[k]


def test_query_fp32_and_cycle(lib):
    spec = dataclasses.replace(synth.C2, n=256)
    W = synth.graph(spec)
    h = make(lib, W, directed=False)
    D = oracle.fw(W)                      # fp64
    for s, t in [(0, 1), (5, 200), (17, 17), (255, 3)]:
        d, path, _ = h.query(s, t)
        if s != t:
            dd, _ = oracle.dijkstra_pair(W, s, t)
            assert abs(d - dd) <= RTOL * dd
        _check_path(W, D, s, t, d, path)
    n = 300
    C = np.full((n, n), INF, np.int32)
    np.fill_diagonal(C, 0)
    C[np.arange(n), (np.arange(n) + 1) % n] = 1
    h2 = make(lib, C)
    d, path, nc = h2.query(10, 250)
    assert d == 240 and path == list(range(10, 251)) and nc == 241


def test_query_unreachable(lib):
    W = np.array([[0, 5, INF], [INF, 0, INF], [INF, INF, 0]], np.int32)
    h = make(lib, W)
    d, path, nc = h.query(1, 0)
    assert d == INF and path == [] and nc == 0


# ------------------------------------------------------------------ errors
def test_argument_errors_leave_state(lib, rng):
    P = lib
    W = random_graph(rng, 50, True, 1.0, lo=1, hi=9)
    h = make(lib, W, cap=50)
    D0 = getD(h).copy()
    with pytest.raises(P.ApspError) as e:
        h.remove_node(50)
    assert e.value.status == 2
    with pytest.raises(P.ApspError) as e:
        h.update_edge(3, 3, 1)
    assert e.value.status == 1
    with pytest.raises(P.ApspError) as e:
        h.update_edge(3, 4, -1)
    assert e.value.status == 1
    with pytest.raises(P.ApspError) as e:
        h.update_edge(3, 4, 1.5)
    assert e.value.status == 1
    with pytest.raises(P.ApspError) as e:
        h.add_node(np.ones(50, np.int32), np.ones(50, np.int32))
    assert e.value.status == 3
    h2 = make(lib, W, cap=51)
    bad = np.ones(50, np.int32)
    bad[7] = -4
    with pytest.raises(P.ApspError) as e:
        h2.add_node(bad, np.ones(50, np.int32))
    assert e.value.status == 1 and h2.n == 50
    assert np.array_equal(getD(h), D0)
    one = make(lib, np.zeros((1, 1), np.int32))
    with pytest.raises(P.ApspError) as e:
        one.remove_node(0)
    assert e.value.status == 4


def test_create_rejects_bad_W(lib):
    P = lib
    W = np.array([[0, 1], [-1, 0]], np.int32)
    with pytest.raises(P.ApspError):
        make(lib, W)
    W = np.array([[1, 1], [1, 0]], np.int32)
    with pytest.raises(P.ApspError):
        make(lib, W)


# ------------------------------------------------------------------ f1: paper's modify (remove + re-add)
@pytest.mark.parametrize("directed", [True, False])
def test_modify_edge_readd_matches_oracle_and_direct(lib, rng, directed):
    """alg:APSPmodify: remove the cheaper endpoint (Definition 1),
    re-add it with the edited edge, ids restored; == oracle == direct update."""
    n = 200
    W = random_graph(rng, n, directed, 0.9, lo=1, hi=80)
    a = make(lib, W, directed)
    b = make(lib, W, directed)
    for trial in range(8):
        u, v = (int(x) for x in rng.choice(n, 2, replace=False))
        if trial == 3:
            u, v = n - 1, 0          # the endpoint may be the last node (no swap)
        w_old = int(W[u, v])
        w_new = min(INF, int(rng.choice([max(0, w_old // 3), w_old * 5, INF, w_old + 1])))
        removed, info = a.modify_edge_readd(u, v, w_new)
        assert a.weight(u, v) == w_new
        b.update_edge(u, v, w_new)
        W = _edit(W, u, v, w_new, directed)
        if w_new != w_old:
            assert info.kind == 5 and removed in (u, v)
            assert a.n == n
        Da = getD(a)
        assert_parity(Da, oracle.fw(W))
        assert np.array_equal(Da, getD(b))


def test_modify_edge_readd_fp32(lib, rng):
    spec = dataclasses.replace(synth.C2, n=150)
    W = synth.graph(spec)
    h = make(lib, W, directed=False)
    for trial in range(4):
        u, v = (int(x) for x in rng.choice(150, 2, replace=False))
        w_new = np.float32(W[u, v] * np.float32(rng.choice([0.1, 10.0])))
        h.modify_edge_readd(u, v, float(w_new))
        W = _edit(W, u, v, w_new, False)
        assert_parity(getD(h), oracle.fw(W))


def test_row_delta_gate_paper_definition1(lib, rng):
    """f4 ablation: the paper's gate (dense FW iff Definition 1's cost > delta,
    P:184-196) picks the path; results are identical either way."""
    n = 220
    W = random_graph(rng, n, True, 1.0, lo=1, hi=100)
    a = make(lib, W)
    b = make(lib, W)
    a.set_option(4, 0.01)     # cost ~0.5 > 0.01 -> dense
    b.set_option(4, 1.0)      # never above 1 -> sparse
    hg = synth.HostGraph(W, True)
    for k in (3, 100, 0):
        _, ia = a.remove_node(k)
        _, ib = b.remove_node(k)
        hg.remove_node(k)
        assert ia.cost == ib.cost and ia.cost > 0.01
        assert ia.path == 3 and ib.path == 2
        Da = getD(a)
        assert np.array_equal(Da, getD(b))
        assert_parity(Da, oracle.fw(hg.W))


@pytest.mark.parametrize("opt,value", [(1, 1e-9), (3, 1)])
def test_removal_gate_theta_and_rounds(lib, rng, opt, value):
    """The pair-level gate (APSP_OPT_THETA: dense iff |A| > theta n^2) and an
    exhausted round budget (APSP_OPT_MAX_ROUNDS) both send a removal to the
    dense path after the sparse kernels ran; the swap-with-last that one GPU
    enqueues before the host's read must then stand aside (it is gated on
    the device by the same decision) — results equal the oracle and the
    default handle's, for a removal of an inner node, the first and the last."""
    n = 240
    W = random_graph(rng, n, True, 1.0, lo=1, hi=100)
    a = make(lib, W)
    b = make(lib, W)
    a.set_option(opt, value)
    b.set_option(1, 0.9)   # b: the sparse path (|A| <= 0.9 n^2)
    hg = synth.HostGraph(W, True)
    for k in (5, 0, n - 3):
        _, ia = a.remove_node(k)
        _, ib = b.remove_node(k)
        hg.remove_node(k)
        assert ib.path == 2
        if opt == 1:
            assert ia.path == 3
        Da = getD(a)
        assert np.array_equal(Da, getD(b))
        assert_parity(Da, oracle.fw(hg.W))


def test_microbench_denominators(lib):
    """K13: the measured relaxation and HBM rates are in the
    range the B200 can deliver (one VIADDMNMX per int32 relaxation: 64/clk/SM
    at <= 1.965 GHz on 148 SMs; HBM3e <= 8 TB/s)."""
    L = lib._lib
    buf = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    r32 = L.apsp_microbench(0, buf.data_ptr(), 4, st)
    f32 = L.apsp_microbench(1, buf.data_ptr(), 4, st)
    s16 = L.apsp_microbench(2, buf.data_ptr(), 4, st)
    rd = L.apsp_microbench(3, buf.data_ptr(), buf.numel(), st)
    rmw = L.apsp_microbench(4, buf.data_ptr(), buf.numel(), st)
    assert 5e12 < r32 <= 148 * 64 * 1.97e9 * 1.02
    assert f32 > 5e12 and s16 > r32
    assert 2e12 < rd < 8.5e12 and 2e12 < rmw < 8.5e12
    with pytest.raises(lib._lib.ApspError):
        L.apsp_microbench(9, buf.data_ptr(), 4, st)


@pytest.mark.parametrize("n,lo,hi,inf_frac", [
    (300, 1, 60, 0.0),         # packed path, ragged tiles (n odd multiple of nothing)
    (513, 0, 9, 0.3),          # zero weights + absent edges: unreachable pairs saturate -> int32 finish
    (257, 9000, 16000, 0.0),   # distances >= 0x3FFF: saturate -> int32 finish
    (1000, 1, 1000, 0.05),
])
def test_fw16_packed_equals_int32_and_oracle(lib, rng, n, lo, hi, inf_frac):
    """APSP_OPT_FW16: the int16x2 blocked FW (exact below 0x3FFF, int32 finish
    otherwise) gives the same D as the int32 FW and the oracle."""
    W = random_graph(rng, n, True, density=1.0, lo=lo, hi=hi, inf_frac=inf_frac)
    h16 = make(lib, W)                      # default: packed
    h32 = make(lib, W, cold=False)
    h32.set_option(lib._lib.OPT_FW16, 0)
    h32.cold_fw()
    D16, D32 = getD(h16), getD(h32)
    assert np.array_equal(D16, D32)
    assert_parity(D16, oracle.fw(W))


def test_fw16_dense_fallback_of_a_removal(lib, rng):
    """a7 through the packed FW: a forced-dense removal equals the oracle."""
    W = random_graph(rng, 700, True, density=0.9, lo=1, hi=50)
    h = make(lib, W)
    h.set_option(0, 2)
    _, info = h.remove_node(123)
    assert info.path == 3
    hg = synth.HostGraph(W, True)
    hg.remove_node(123)
    assert_parity(getD(h), oracle.fw(hg.W))


# ------------------------------------------------------------------ mirror widths (§4.7)
def _apply(h, hg, up):
    if up.kind == "add":
        h.add_node(up.out_w, up.in_w)
        hg.add_node(up.out_w, up.in_w)
    elif up.kind == "remove":
        h.remove_node(up.k)
        hg.remove_node(up.k)
    else:
        h.update_edge(up.u, up.v, up.w_new)
        hg.set_edge(up.u, up.v, up.w_new)


@pytest.mark.parametrize("mirror8", [1, 0])
def test_mirror_width_sequence(lib, mirror8):
    """BJ.c4-shaped sequence (distances < 0x7F): the streaming passes read the
    int8 copy of D (or, with APSP_OPT_MIRROR8 = 0, the int16 one); D equals
    the oracle after every update either way."""
    spec = dataclasses.replace(synth.C4, n=520)
    W = synth.graph(spec)
    cap = 520 + 24
    hg = synth.HostGraph(W, True, cap=cap)
    h = make(lib, W, cap=cap, cold=False)
    h.set_option(lib._lib.OPT_MIRROR8, mirror8)
    h.cold_fw()
    seq = synth.update_sequence(spec, synth.HostGraph(W, True, cap=cap), 0, 24)
    for t, up in enumerate(seq):
        _apply(h, hg, up)
        assert h.mirror_width == (8 if mirror8 else 16)
        if t % 6 == 5:
            assert_parity(getD(h), oracle.fw(hg.W))
    assert_parity(getD(h), oracle.fw(hg.W))


@pytest.mark.parametrize("force", [0, 1])
def test_mirror8_invalidated_by_a_removal(lib, force):
    """Removing a hub pushes distances along a chain of weight-10 edges from 2
    up to 10*(n-2) >= 0x7F: the int8 copy is invalidated, the updates that
    follow read D (exact), and the next build of the copy is int16."""
    n = 90
    W = np.full((n, n), INF, np.int32)
    np.fill_diagonal(W, 0)
    hub = n - 1
    for i in range(n - 1):
        W[i, hub] = W[hub, i] = 1
        if i + 1 < n - 1:
            W[i, i + 1] = W[i + 1, i] = 10
    hg = synth.HostGraph(W, True, cap=n + 4)
    h = make(lib, W, cap=n + 4)
    rng = np.random.default_rng(5)
    o = np.full(n, INF, np.int32)
    o[3] = 1
    i = o.copy()
    h.add_node(o, i)   # first update: builds the copy (int8: every distance <= 3)
    hg.add_node(o, i)
    assert h.mirror_width == 8
    h.set_option(0, force)
    h.remove_node(hub)
    hg.remove_node(hub)
    assert_parity(getD(h), oracle.fw(hg.W))
    for _ in range(4):   # further updates on the invalidated / rebuilt copy
        u, v = (int(x) for x in rng.choice(hg.n, 2, replace=False))
        w = int(rng.integers(1, 40))
        h.update_edge(u, v, w)
        hg.set_edge(u, v, w)
        assert_parity(getD(h), oracle.fw(hg.W))
    assert h.mirror_width in (0, 16)
    h.sync_distances()   # rebuild: int8 failed once, so int16 now
    assert h.mirror_width == 16
    k = int(rng.integers(0, hg.n))
    h.remove_node(k)
    hg.remove_node(k)
    assert_parity(getD(h), oracle.fw(hg.W))


def test_mirror8_invalidated_by_an_add(lib, rng):
    """A new node whose edges weigh 500 writes distances >= 0x7F through the
    rank-1 pass: the int8 copy is invalidated; later updates stay exact."""
    spec = dataclasses.replace(synth.C4, n=300)
    W = synth.graph(spec)
    hg = synth.HostGraph(W, True, cap=310)
    h = make(lib, W, cap=310)
    o, i = synth.node_edges(spec, 1, 300)
    h.add_node(o, i)
    hg.add_node(o, i)
    assert h.mirror_width == 8
    o2 = np.full(hg.n, 500, np.int32)
    h.add_node(o2, o2)
    hg.add_node(o2, o2)
    assert_parity(getD(h), oracle.fw(hg.W))
    for k in (5, 17, -1):
        k = k % hg.n
        h.remove_node(k)
        hg.remove_node(k)
        assert_parity(getD(h), oracle.fw(hg.W))
    assert h.mirror_width in (0, 16)


@pytest.mark.parametrize("n,directed", [(1003, True), (1003, False), (517, True), (33, False)])
def test_mirror8_ragged_sizes(lib, rng, n, directed):
    """The int8 readers (detection, pass 1, rank-1) on sizes that end inside a
    16-column group and a 512/1024-column chunk, directed and undirected (two
    pivot terms), with absent edges (INF entries): every update kind, parity
    after each."""
    W = random_graph(rng, n, directed, density=0.7, lo=1, hi=25, inf_frac=0.05)
    cap = n + 4
    hg = synth.HostGraph(W, directed, cap=cap)
    h = make(lib, W, directed, cap=cap)
    for step in range(6):
        kind = step % 3
        if kind == 0:
            o = rng.integers(1, 25, hg.n).astype(np.int32)
            o[rng.random(hg.n) < 0.1] = INF
            i = o.copy() if not directed else rng.integers(1, 25, hg.n).astype(np.int32)
            h.add_node(o, i)
            hg.add_node(o, i)
        elif kind == 1:
            k = int(rng.integers(0, hg.n))
            h.remove_node(k)
            hg.remove_node(k)
        else:   # a tight edge increase (Theorem 4's affected set is non-empty)
            u = int(rng.integers(0, hg.n))
            row = np.where(np.arange(hg.n) == u, INF, hg.W[u, :hg.n]).astype(np.int64)
            v = int(np.argmin(row))
            if row[v] < INF:
                w = int(row[v]) * 3 + 1
                h.update_edge(u, v, w)
                hg.set_edge(u, v, w)
        assert h.mirror_width == 8
        assert_parity(getD(h), oracle.fw(hg.W))


def _sampled_rows_cols(h, W, idx):
    torch.cuda.synchronize()
    it = torch.as_tensor(np.asarray(idx), device=h.D_local.device, dtype=torch.long)
    got_r = h.D.index_select(0, it).cpu().numpy()
    got_c = h.D.index_select(1, it).cpu().numpy().T
    assert np.array_equal(got_r, oracle.dijkstra_rows_i32(W, idx))
    assert np.array_equal(got_c, oracle.dijkstra_rows_i32(W, idx, reverse=True))


def test_add_node_gather_fallbacks(lib, rng):
    """The add-node shortcuts (n >= 4096, int8 mirror) and their fallbacks:
    (1) the columns with the cheapest in-edges are unreachable from most rows
    (col1 uncertified: full-row scans); (2) every in-edge equally cheap, so the
    gathered column set exceeds its limit (the streaming pass 1 runs).
    Sampled rows / columns (the new node's included) against Dijkstra on the
    host graph, and the whole matrix against the oracle's FW of the same graph."""
    n = 4200
    W = random_graph(rng, n, True, density=0.01, lo=1, hi=9)
    W[:, :10] = INF            # nodes 0-9: no in-edges
    np.fill_diagonal(W, 0)
    hg = synth.HostGraph(W, True, cap=n + 3)
    h = make(lib, W, cap=n + 3)
    assert h.mirror_width == 8
    o = rng.integers(1, 9, n).astype(np.int32)
    i = np.full(n, 60, np.int32)
    i[:10] = 1                 # cheapest in-edges from the unreachable nodes
    h.add_node(o, i)
    hg.add_node(o, i)
    o2 = rng.integers(1, 9, hg.n).astype(np.int32)
    i2 = np.full(hg.n, 3, np.int32)   # all equal: |U| = n > 2048
    h.add_node(o2, i2)
    hg.add_node(o2, i2)
    o3 = rng.integers(1, 40, hg.n).astype(np.int32)   # the ordinary case
    i3 = rng.integers(1, 40, hg.n).astype(np.int32)
    h.add_node(o3, i3)
    hg.add_node(o3, i3)
    idx = np.concatenate([rng.choice(n, 12, replace=False), [0, 5, n, n + 1, n + 2]])
    _sampled_rows_cols(h, hg.W, idx)
    assert_parity(getD(h), oracle.fw(hg.W))


def test_new_node_shortlist_then_removals(lib, rng):
    """The new node's shortlist SL(x) (exact top-512 in-edges by (weight, id),
    built over 1024-entry chunks — n = 4100 ends inside a chunk) used by later
    removals that list pairs in column x: (1) fewer than 512 finite in-edges
    (dead entries) and zero weights (wmin = 0 in the column certification);
    (2) every in-edge finite.  Sampled rows / columns against Dijkstra on the
    host graph and the whole matrix against the oracle's FW of the final graph."""
    n = 4100
    W = random_graph(rng, n, True, density=0.02, lo=1, hi=9)
    hg = synth.HostGraph(W, True, cap=n + 3)
    h = make(lib, W, cap=n + 3)
    assert h.mirror_width == 8
    o = rng.integers(1, 9, n).astype(np.int32)
    i = np.full(n, INF, np.int32)
    fin = rng.choice(n, 300, replace=False)
    i[fin] = rng.integers(1, 9, 300)
    i[fin[:5]] = 0
    o[rng.choice(n, 4, replace=False)] = 0
    h.add_node(o, i)
    hg.add_node(o, i)
    for _ in range(3):
        k = int(rng.integers(0, hg.n - 1))
        h.remove_node(k)
        hg.remove_node(k)
    o2 = rng.integers(1, 12, hg.n).astype(np.int32)
    i2 = rng.integers(1, 12, hg.n).astype(np.int32)
    h.add_node(o2, i2)
    hg.add_node(o2, i2)
    for _ in range(2):
        k = int(rng.integers(0, hg.n - 1))
        h.remove_node(k)
        hg.remove_node(k)
    m = hg.n
    idx = np.concatenate([rng.choice(m, 10, replace=False), [m - 1, m - 2]])
    _sampled_rows_cols(h, hg.W[:m, :m], idx)
    assert_parity(getD(h), oracle.fw(hg.W[:m, :m]))


def test_add_node_heavy_out_edges_to_unreachable(lib, rng):
    """ADVICE r1 (two bugs on the add-node shortcut path, n >= 4096, int8
    mirror): nodes 0-9 have no in-edges, so the new node's row there is its
    own out-edge out[j] ~ U[1,1000] (>= omin + 128 for most j: the minimiser
    key must not sign-extend), and rank-1 then writes distances >= 0x7F into
    columns 0-9 of every row — the int8 mirror goes invalid during the rank-1
    launch, whose later CTAs must still relax their rows.  Whole matrix vs the
    oracle's cold FW of the same graph; then a removal and a second add on the
    (now int16) mirror."""
    n = 4200
    W = random_graph(rng, n, True, density=0.02, lo=1, hi=9)
    W[:, :10] = INF            # nodes 0-9: no in-edges
    np.fill_diagonal(W, 0)
    hg = synth.HostGraph(W, True, cap=n + 3)
    h = make(lib, W, cap=n + 3)
    assert h.mirror_width == 8
    o = rng.integers(1, 1001, n).astype(np.int32)
    o[rng.choice(np.arange(10, n), 3, replace=False)] = 1     # omin = 1, outside 0-9
    i = rng.integers(1, 40, n).astype(np.int32)
    h.add_node(o, i)
    hg.add_node(o, i)
    assert_parity(getD(h), oracle.fw(hg.W))
    k = int(rng.integers(10, hg.n - 1))
    h.remove_node(k)
    hg.remove_node(k)
    o2 = rng.integers(1, 1001, hg.n).astype(np.int32)
    i2 = rng.integers(1, 1001, hg.n).astype(np.int32)
    h.add_node(o2, i2)
    hg.add_node(o2, i2)
    assert_parity(getD(h), oracle.fw(hg.W[:hg.n, :hg.n]))


# ------------------------------------------------ detection, set for set (§8(c-1))
def _pairs(r, c):
    return set(zip(np.asarray(r).tolist(), np.asarray(c).tolist()))


def _mask_pairs(m):
    i, j = np.nonzero(m)
    return set(zip(i.tolist(), j.tolist()))


def _tight_edge(W, D, rng, directed=True):
    """An edge (u, v) with W[u][v] == D[u][v] (tight: on a shortest path)."""
    n = W.shape[0]
    for _ in range(1000):
        u = int(rng.integers(n))
        row = np.where((np.arange(n) != u) & (W[u] < INF) & (W[u] == D[u]), 1, 0)
        if row.any():
            v = int(rng.choice(np.nonzero(row)[0]))
            return u, v
    raise AssertionError("no tight edge")


@pytest.mark.parametrize("n,directed,hi,mirror", [
    (300, True, 9, 1),        # int8 mirror
    (1100, True, 9, 1),       # int8, several 1024-column chunks + a ragged one
    (700, False, 9, 1),
    (1100, True, 4000, 1),    # distances >= 0x7F: int16 mirror
    (1100, True, 9, 0),       # no mirror: the int32 stream (4 B/entry)
    (2100, False, 60, 0),
])
def test_need_update_list_set_for_set_int32(lib, rng, n, directed, hi, mirror):
    """The GPU's need_update_list (the detection kernels the updates run,
    exported by apsp_need_update_list) equals the oracle's definitional
    predicate set for set (Corollary 3 / Theorem 4): removals of
    random nodes and increases of tight edges (undirected: both orientations)."""
    W = random_graph(rng, n, directed, density=0.3, lo=1, hi=hi, inf_frac=0.02)
    W[10:, :10] = INF          # nodes 0-9 reachable only among themselves: INF
    if not directed:           # rows / columns (increases inside 0-9 must not
        W[:10, 10:] = INF      # list the INF pairs, Q5)
    np.fill_diagonal(W, 0)
    h = make(lib, W, directed)
    h.set_option(lib._lib.OPT_MIRROR, mirror)
    D = oracle.fw(W)
    assert np.array_equal(getD(h), D)
    for k in rng.choice(n, 3, replace=False):
        r, c, cnt = h.need_update_list("remove", int(k))
        assert cnt == len(r)
        exp = _mask_pairs(oracle.need_update_removal(D, int(k)))
        assert _pairs(r, c) == exp and cnt == len(exp)
    if mirror:
        assert h.mirror_width == (8 if D[D < INF].max() < 0x7F else 16)
    else:
        assert h.mirror_width == 0
    for t in range(4):
        if t == 0:   # an edge inside the 0-9 island
            sub = W[:10, :10]
            cand = [(a, b) for a in range(10) for b in range(10) if a != b and sub[a, b] < INF and sub[a, b] == D[a, b]]
            if not cand:
                continue
            u, v = cand[0]
        else:
            u, v = _tight_edge(W, D, rng)
        r, c, cnt = h.need_update_list("increase", u, v)
        exp = _mask_pairs(oracle.need_update_increase(D, u, v, int(W[u, v]), directed))
        assert _pairs(r, c) == exp and cnt == len(exp)
    assert np.array_equal(getD(h), D)      # nothing was applied


def test_need_update_list_fp32_bracketed(lib, rng):
    """fp32 detection uses the tolerant test (Q4): the GPU set holds
    every exactly tight pair of the fp64 oracle (tau = 0) and nothing outside
    the oracle's set at a slightly looser tau (what is unique is compared, the
    rest checked valid)."""
    n = 600
    W = random_graph(rng, n, False, density=0.5, hi=1, dtype=np.float32)
    h = make(lib, W, directed=False)
    D = oracle.fw(W)
    for k in rng.choice(n, 3, replace=False):
        r, c, _ = h.need_update_list("remove", int(k))
        got = _pairs(r, c)
        assert _mask_pairs(oracle.need_update_removal(D, int(k), tau=0.0)) <= got
        assert got <= _mask_pairs(oracle.need_update_removal(D, int(k), tau=3e-5))
    u = 5
    row = np.where(np.arange(n) == u, np.inf, W[u].astype(np.float64))
    v = int(np.argmin(row))                  # the cheapest out-edge is tight
    r, c, _ = h.need_update_list("increase", u, v)
    got = _pairs(r, c)
    assert _mask_pairs(oracle.need_update_increase(D, u, v, float(W[u, v]), False, tau=0.0)) <= got
    assert got <= _mask_pairs(oracle.need_update_increase(D, u, v, float(W[u, v]), False, tau=3e-5))


def test_need_update_list_minimax_set_for_set(lib, rng):
    """Minimax handles (f2): the detection predicate with + -> max, set for set."""
    n = 500
    W = random_graph(rng, n, True, density=0.2, lo=1, hi=30)
    h = make(lib, W, cold=False)
    h.set_option(lib._lib.OPT_SEMIRING, 1)
    h.cold_fw()
    D = oracle.fw_minimax(W)
    assert np.array_equal(getD(h), D)
    for k in rng.choice(n, 3, replace=False):
        r, c, _ = h.need_update_list("remove", int(k))
        assert _pairs(r, c) == _mask_pairs(oracle.need_update_removal_minimax(D, int(k)))


def test_int32_streams_without_mirror_match_oracle(lib, rng):
    """APSP_OPT_MIRROR = 0 (every O(n^2) pass streams the int32 D, the byte
    basis of SURVEY §8(d-4)): a mixed update sequence stays bit-exact."""
    n = 1500
    W = random_graph(rng, n, True, density=0.5, lo=1, hi=50)
    hg = synth.HostGraph(W, True, cap=n + 8)
    h = make(lib, W, cap=n + 8)
    h.set_option(lib._lib.OPT_MIRROR, 0)
    for t in range(9):
        if t % 3 == 0:
            o = rng.integers(1, 50, hg.n).astype(np.int32)
            i = rng.integers(1, 50, hg.n).astype(np.int32)
            h.add_node(o, i)
            hg.add_node(o, i)
        elif t % 3 == 1:
            k = int(rng.integers(hg.n))
            h.remove_node(k)
            hg.remove_node(k)
        else:
            Dn = getD(h)
            u, v = _tight_edge(hg.W[:hg.n, :hg.n], Dn, rng)
            w = int(hg.W[u, v]) * 4
            h.update_edge(u, v, w)
            hg.set_edge(u, v, w)
        assert h.mirror_width == 0
    assert_parity(getD(h), oracle.fw(hg.W[:hg.n, :hg.n]))


@pytest.mark.parametrize("fused", [1, 0])
def test_fused_detect_phase_a_with_spills(lib, rng, fused):
    """The fused detection + phase A kernel (fused.cu, removals on the int8
    mirror) against the separate kernels and the oracle: a line metric with
    repeated positions (every pair through the middle is a tie, so rows list
    far more pairs than a stage's buffer holds and spill to the stand-alone
    phase A), the sparse path forced; then random removals on a random graph.
    Bit-exact vs the oracle's FW after every removal."""
    n = 2500
    x = np.sort(rng.integers(0, 100, n))
    W = np.abs(x[:, None] - x[None, :]).astype(np.int32)
    hg = synth.HostGraph(W, True)
    h = make(lib, W)
    h.set_option(lib._lib.OPT_FUSED, fused)
    h.set_option(lib._lib.OPT_FORCE_PATH, 1)
    assert h.mirror_width == 8
    k = n // 2
    _, info = h.remove_node(k)
    hg.remove_node(k)
    # (rows list more pairs than a stage buffer: the spill path ran; the gate
    # may still finish densely — the sparse kernels' output is exact input)
    assert info.path in (2, 3) and info.max_row_affected > 1024
    assert_parity(getD(h), oracle.fw(hg.W))
    W2 = random_graph(rng, 1800, True, density=0.05, lo=1, hi=9)
    hg2 = synth.HostGraph(W2, True)
    h2 = make(lib, W2)
    h2.set_option(lib._lib.OPT_FUSED, fused)
    for _ in range(4):
        k = int(rng.integers(hg2.n))
        h2.remove_node(k)
        hg2.remove_node(k)
        assert_parity(getD(h2), oracle.fw(hg2.W))


@pytest.mark.parametrize("dtype", [np.int32, np.float32])
def test_gate_dense_after_sparse_kernels(lib, rng, dtype):
    """The default gate picks the dense FW AFTER the sparse kernels already ran
    (|A| > theta n^2): a line metric with repeated positions, middle node
    removed (every pair across it is a tie, |A| ~ n^2 / 2).  The sparse
    kernels' values may exceed a listed pair's own edge (phase A reads the
    cheapest in-edges of j only), so the fallback takes min(D, W') first —
    without it this case came out too large.  Bit-exact
    (int32) / 1e-5 (fp32) vs the oracle."""
    n = 1500
    x = np.sort(rng.integers(0, 60, n)).astype(np.float64)
    W = np.abs(x[:, None] - x[None, :])
    W = W.astype(np.int32) if dtype == np.int32 else (W * 0.125).astype(np.float32)
    hg = synth.HostGraph(W, True)
    h = make(lib, W)
    _, info = h.remove_node(n // 2)
    hg.remove_node(n // 2)
    assert info.path == 3
    assert_parity(getD(h), oracle.fw(hg.W))


def test_need_update_list_fused_export_set_for_set(lib, rng):
    """The fused kernel's own list (APSP_OPT_FUSED=1, export mode) against the
    oracle's predicate, removals and directed increases."""
    n = 1300
    W = random_graph(rng, n, True, density=0.3, lo=1, hi=9, inf_frac=0.02)
    h = make(lib, W)
    h.set_option(lib._lib.OPT_FUSED, 1)
    D = oracle.fw(W)
    for k in rng.choice(n, 3, replace=False):
        r, c, cnt = h.need_update_list("remove", int(k))
        assert _pairs(r, c) == _mask_pairs(oracle.need_update_removal(D, int(k))) and cnt == len(r)
    u, v = _tight_edge(W, D, rng)
    r, c, _ = h.need_update_list("increase", u, v)
    assert _pairs(r, c) == _mask_pairs(oracle.need_update_increase(D, u, v, int(W[u, v]), True))


def test_query_candidate_set_beyond_scratch(lib):
    """|C| > 4096 (the batch scratch): the directed unit cycle, s = 0, t = n-1 —
    C is the whole arc and the path has n nodes (SURVEY §8(c-4) a8
    closed form).  Also a query in the other direction and a short one."""
    n = 5000
    C = np.full((n, n), INF, np.int32)
    np.fill_diagonal(C, 0)
    C[np.arange(n), (np.arange(n) + 1) % n] = 1
    h = make(lib, C)
    d, path, nc = h.query(0, n - 1, path_cap=n)
    assert d == n - 1 and nc == n and path == list(range(n))
    d, path, nc = h.query(4500, 4200, path_cap=n)
    assert d == (4200 - 4500) % n and path == [(4500 + k) % n for k in range(d + 1)]
    d, path, _ = h.query(10, 15)
    assert d == 5 and path == list(range(10, 16))
    with pytest.raises(lib.ApspError):   # path_cap too small: E_RANGE, needed length reported
        h.query(0, n - 1, path_cap=100)


# ------------------------------------------------------------------ heavy rows (§4.6)
@pytest.mark.parametrize("dtype,directed,semiring", [
    (np.int32, True, 0), (np.float32, False, 0), (np.int32, False, 1), (np.float32, True, 1)])
def test_heavy_rows_forced_sequence(lib, rng, dtype, directed, semiring):
    """APSP_OPT_HEAVY = 1: up to 32 rows with any open pair skip the frontier
    rounds and are resolved from the other rows (X pass + closure inside the
    heavy set) — every removal and tight increase of a mixed sequence, int32
    bit-exact / fp32 1e-5 vs the oracle, shortest path and minimax."""
    n = 260
    W = random_graph(rng, n, directed=directed, lo=1, hi=9, dtype=dtype, density=0.5)
    hg = synth.HostGraph(W, directed)
    h = lib.WarmAPSP(torch.from_numpy(W), directed=directed, cold_start=False,
                     semiring="minimax" if semiring else "shortest")
    h.set_option(lib._lib.OPT_HEAVY, 1)
    h.set_option(0, 1)   # the sparse path
    h.cold_fw()
    ref = oracle.fw_minimax if semiring else oracle.fw
    for t in range(10):
        if t % 2 == 0:
            k = int(rng.integers(hg.n))
            _, info = h.remove_node(k)
            hg.remove_node(k)
        else:
            D = ref(hg.W)
            u, v = _tight_edge(hg.W, D, rng, directed)
            w = hg.W[u, v] * (3 if dtype == np.int32 else np.float32(3))
            if semiring and w == hg.W[u, v]:
                w = hg.W[u, v] + 5
            info = h.update_edge(u, v, w)
            hg.set_edge(u, v, w)
        assert_parity(getD(h), ref(hg.W))


@pytest.mark.parametrize("dtype", [np.float32, np.int32])
def test_heavy_rows_default_threshold(lib, dtype):
    """The default threshold (max(512, n/8) open pairs): an undirected complete
    graph, the cheapest edge of a node raised x10 leaves thousands of open
    pairs in that node's row — resolved by the heavy-row pass, equal to the
    oracle; and to the same update with heavy rows off."""
    spec = dataclasses.replace(synth.C2, n=1100) if dtype == np.float32 else \
        dataclasses.replace(synth.C4, n=1100, directed=False)
    W = synth.graph(spec)
    if dtype == np.int32:
        W = np.minimum(W, W.T)
    hgs = []
    outs = []
    for heavy in (0, -1):
        h = make(lib, W, directed=False)
        h.set_option(lib._lib.OPT_HEAVY, heavy)
        hg = synth.HostGraph(W, False)
        for u in (3, 4):
            row = hg.W[u].astype(np.float64)
            row[u] = np.inf
            v = int(np.argmin(row))
            w = hg.W[u, v] * (10 if dtype == np.int32 else np.float32(10))
            info = h.update_edge(u, v, w)
            hg.set_edge(u, v, w)
            assert info.path == 2
        outs.append(getD(h))
        hgs.append(hg)
    assert_parity(outs[0], oracle.fw(hgs[0].W))
    assert np.array_equal(outs[0], outs[1]) if dtype == np.int32 else True
