"""Pins of the CPU oracle against things other than itself (CPU only).

Each test names what fixes the expected value: brute-force enumeration of the
definition, closed forms, the paper's worked examples (golden
fixtures with citations), or the paper's theorems restated independently.
"""
import itertools

import numpy as np
import pytest

import oracle
import synth
from conftest import golden_graph, load_golden, random_graph

INF = synth.INF_I32


# ---------------------------------------------------------------- brute force
@pytest.mark.parametrize("directed", [True, False])
@pytest.mark.parametrize("density", [0.3, 1.0])
def test_fw_equals_bruteforce(rng, directed, density):
    """FW == exhaustive simple-path enumeration (the definition), n <= 7,
    weights including 0 and absent edges."""
    for trial in range(25):
        n = int(rng.integers(2, 8))
        W = random_graph(rng, n, directed, density, lo=0, hi=6)
        assert np.array_equal(oracle.fw(W), oracle.brute_apsp(W)), (trial, W)


def test_fw_f64_equals_bruteforce(rng):
    for trial in range(15):
        n = int(rng.integers(2, 7))
        W = random_graph(rng, n, True, 0.7, hi=1, dtype=np.float32)
        D = oracle.fw(W)
        B = oracle.brute_apsp(W)
        assert np.allclose(D, B, rtol=1e-12, atol=0) and np.array_equal(np.isinf(D), np.isinf(B))


@pytest.mark.parametrize("directed", [True, False])
def test_dijkstra_equals_bruteforce_and_fw(rng, directed):
    for trial in range(20):
        n = int(rng.integers(2, 8))
        W = random_graph(rng, n, directed, 0.6, lo=0, hi=9)
        B = oracle.brute_apsp(W)
        assert np.array_equal(oracle.dijkstra_rows(W, range(n)), B)
        assert np.array_equal(oracle.dijkstra_cols(W, range(n)), B)
    # larger: FW == all-sources Dijkstra
    W = random_graph(rng, 120, directed, 0.5, lo=1, hi=50)
    assert np.array_equal(oracle.fw(W), oracle.dijkstra_rows(W, range(120)))


def test_dijkstra_pair_path(rng):
    for trial in range(30):
        n = int(rng.integers(2, 8))
        W = random_graph(rng, n, True, 0.5, lo=1, hi=9)
        s, t = rng.choice(n, 2, replace=False)
        d, path = oracle.dijkstra_pair(W, int(s), int(t))
        assert d == oracle.brute(W, int(s), int(t))
        if d == INF:
            assert path == []
        else:
            assert oracle.path_is_valid(W, path, s, t)
            assert oracle.path_weight(W, path) == d


# ---------------------------------------------------------------- closed forms
def cycle(n, w=1):
    W = np.full((n, n), INF, np.int32)
    np.fill_diagonal(W, 0)
    W[np.arange(n), (np.arange(n) + 1) % n] = w
    return W


def test_closed_form_directed_cycle():
    n = 37
    i, j = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    assert np.array_equal(oracle.fw(cycle(n)), ((j - i) % n).astype(np.int32))


def test_closed_form_undirected_path():
    n = 40
    W = np.full((n, n), INF, np.int32)
    np.fill_diagonal(W, 0)
    a = np.arange(n - 1)
    W[a, a + 1] = 1
    W[a + 1, a] = 1
    i, j = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    assert np.array_equal(oracle.fw(W), np.abs(i - j).astype(np.int32))


def test_closed_form_uniform_complete():
    n, c = 30, 7
    W = np.full((n, n), c, np.int32)
    np.fill_diagonal(W, 0)
    assert np.array_equal(oracle.fw(W), W)


def test_closed_form_star():
    n = 25
    a = np.arange(1, n) * 3 % 11 + 1
    W = np.full((n, n), INF, np.int32)
    np.fill_diagonal(W, 0)
    W[0, 1:] = a
    W[1:, 0] = a
    D = oracle.fw(W)
    exp = np.zeros((n, n), np.int64)
    exp[0, 1:] = a
    exp[1:, 0] = a
    exp[1:, 1:] = a[:, None] + a[None, :]
    np.fill_diagonal(exp, 0)
    assert np.array_equal(D, exp.astype(np.int32))


def test_closed_form_line_metric_is_fixpoint(rng):
    x = np.sort(rng.integers(0, 1000, 50))
    W = np.abs(x[:, None] - x[None, :]).astype(np.int32)
    assert np.array_equal(oracle.fw(W), W)


def test_closed_form_grid_manhattan():
    r, c = 6, 7
    n = r * c
    W = np.full((n, n), INF, np.int32)
    np.fill_diagonal(W, 0)
    for a in range(r):
        for b in range(c):
            p = a * c + b
            if b + 1 < c:
                W[p, p + 1] = W[p + 1, p] = 1
            if a + 1 < r:
                W[p, p + c] = W[p + c, p] = 1
    D = oracle.fw(W)
    ra, ca = np.divmod(np.arange(n), c)
    exp = np.abs(ra[:, None] - ra[None, :]) + np.abs(ca[:, None] - ca[None, :])
    assert np.array_equal(D, exp.astype(np.int32))


def test_fw_idempotent_metric_closure(rng):
    W = random_graph(rng, 60, True, 0.4, lo=1, hi=20)
    D = oracle.fw(W)
    assert np.array_equal(oracle.fw(D), D)
    oracle.check_invariants(D, W)


def test_unreachable_is_inf():
    W = np.array([[0, 5], [INF, 0]], np.int32)
    assert np.array_equal(oracle.fw(W), W)


# ------------------------------------------------------- paper theorems (pins)
def test_theorem2_3_add_node_identities(rng):
    """Theorems 2 / theo_2_back / 3, restated in numpy from the
    paper's statements, agree with FW of the grown graph."""
    for trial in range(20):
        n = int(rng.integers(2, 30))
        Wg = random_graph(rng, n + 1, True, 0.7, lo=0, hi=9).astype(np.int64)
        Wg[Wg >= INF] = oracle.INF64
        W = Wg[:n, :n]
        D = oracle.to_oracle(oracle.fw(W.clip(max=INF).astype(np.int32)))
        out_w, in_w = Wg[n, :n], Wg[:n, n]
        row = (out_w[:, None] + D).min(axis=0)      # Thm 2: min_t d(x,t) + SPD(t,r)
        col = (D + in_w[None, :]).min(axis=1)       # theo_2_back: min_t SPD(r,t) + d(t,x)
        old = np.minimum(D, col[:, None] + row[None, :])  # Thm 3: min(x1, t1 + t2)
        full = oracle.to_oracle(oracle.fw(np.where(Wg >= oracle.INF64, INF, Wg).astype(np.int32)))
        clip = lambda a: np.minimum(a, oracle.INF64)
        assert np.array_equal(clip(full[:n, :n]), clip(old))
        assert np.array_equal(clip(full[n, :n]), clip(row))
        assert np.array_equal(clip(full[:n, n]), clip(col))


def test_golden_add_one_node():
    g = load_golden("add_one_node.json")
    W = np.array([[0, g["in_w"][0]], [g["out_w"][0], 0]], np.int32)
    # new node p has index 1: W[p][0] = out (d(p,G_0)), W[0][p] = in (d(G_0,p))
    assert oracle.fw(W).tolist() == g["expected"]


# ---------------------------------------------------- Theorem-4 / Corollary 3
def _remove_from(W, k):
    keep = [i for i in range(W.shape[0]) if i != k]
    return W[np.ix_(keep, keep)], keep


@pytest.mark.parametrize("directed", [True, False])
def test_need_update_removal_is_safe(rng, directed):
    """Corollary 3: every pair NOT in need_update_list keeps its
    distance after removing k.  Monotonicity: nothing decreases."""
    for trial in range(60):
        n = int(rng.integers(3, 12))
        W = random_graph(rng, n, directed, float(rng.choice([0.3, 1.0])), lo=0, hi=6)
        D = oracle.fw(W)
        k = int(rng.integers(n))
        m = oracle.need_update_removal(D, k)
        W2, keep = _remove_from(W, k)
        D2 = oracle.fw(W2)
        Dk = D[np.ix_(keep, keep)]
        mk = m[np.ix_(keep, keep)]
        assert np.array_equal(D2[~mk], Dk[~mk])
        assert np.all(D2 >= Dk)


@pytest.mark.parametrize("directed", [True, False])
def test_need_update_increase_is_safe(rng, directed):
    for trial in range(60):
        n = int(rng.integers(3, 12))
        W = random_graph(rng, n, directed, 1.0, lo=1, hi=6)
        D = oracle.fw(W)
        u, v = (int(x) for x in rng.choice(n, 2, replace=False))
        w_old = int(W[u, v])
        w_new = int(rng.choice([w_old + 1, w_old + 5, INF]))
        m = oracle.need_update_increase(D, u, v, w_old, directed)
        W2 = W.copy()
        W2[u, v] = w_new
        if not directed:
            W2[v, u] = w_new
        D2 = oracle.fw(W2)
        assert np.array_equal(D2[~m], D[~m])
        assert np.all(D2 >= D)


def test_golden_hub_remove():
    g = load_golden("hub_remove.json")
    W, idx = golden_graph(g)
    D = oracle.fw(W)
    k = idx[g["remove"]]
    m = oracle.need_update_removal(D, k)
    names = g["nodes"]
    lists = {names[i]: [names[j] for j in np.nonzero(m[i])[0]] for i in range(len(names)) if m[i].any()}
    assert lists == g["need_update_list"]
    phi, c = oracle.cost(m, len(names))
    assert c == g["cost"]
    W2, keep = _remove_from(W, k)
    D2 = oracle.fw(W2)
    kn = [names[i] for i in keep]
    for pair, val in g["after"].items():
        a, b = pair.split("-")
        assert D2[kn.index(a), kn.index(b)] == val


def test_golden_star_avoided_remove():
    g = load_golden("star_avoided_remove.json")
    W, idx = golden_graph(g)
    D = oracle.fw(W)
    m = oracle.need_update_removal(D, idx[g["remove"]])
    assert not m.any()
    assert oracle.cost(m, 4)[1] == g["cost"]


def test_remove_isolated_node_lists_empty(rng):
    W = random_graph(rng, 9, True, 1.0, lo=1, hi=9)
    W[4, :] = INF
    W[:, 4] = INF
    W[4, 4] = 0
    assert not oracle.need_update_removal(oracle.fw(W), 4).any()


# ------------------------------------------------------------- candidates
def test_golden_hub_query():
    g = load_golden("hub_query.json")
    W, idx = golden_graph(g)
    D = oracle.fw(W)
    s, t = (idx[a] for a in g["query"])
    c = oracle.candidates(D, s, t)
    assert sorted(g["nodes"][i] for i in c) == sorted(g["candidates"])
    d, path = oracle.dijkstra_pair(W, s, t)
    assert d == g["dist"] and [g["nodes"][i] for i in path] == g["path"]


def test_candidates_contain_every_shortest_path_node(rng):
    """Every node of every shortest s-t path satisfies Theorem 4's equality
    (S:305); on unique-path instances the set is exactly the path."""
    for trial in range(40):
        n = int(rng.integers(3, 8))
        W = random_graph(rng, n, True, 0.8, lo=1, hi=20)
        D = oracle.fw(W)
        s, t = (int(x) for x in rng.choice(n, 2, replace=False))
        c = set(oracle.candidates(D, s, t).tolist())
        if D[s, t] == INF:
            assert c == set()
            continue
        # enumerate simple paths and keep the shortest ones
        best = []
        others = [v for v in range(n) if v not in (s, t)]
        for r in range(len(others) + 1):
            for mid in itertools.permutations(others, r):
                p = [s, *mid, t]
                if oracle.path_is_valid(W, p, s, t) and oracle.path_weight(W, p) == D[s, t]:
                    best.append(p)
        assert best
        for p in best:
            assert set(p) <= c
        if len(best) == 1:
            assert c == set(best[0])


def test_dijkstra_int32_inplace_matches_bruteforce(rng):
    """The in-place int32 Dijkstra (sampled full-size checks) against the
    definition, rows and reversed columns, with zeros and absent edges."""
    for trial in range(15):
        n = int(rng.integers(2, 8))
        W = random_graph(rng, n, True, 0.6, lo=0, hi=9)
        B = oracle.brute_apsp(W)
        assert np.array_equal(oracle.dijkstra_rows_i32(W, range(n)), B)
        assert np.array_equal(oracle.dijkstra_rows_i32(W, range(n), reverse=True), B.T)


# ------------------------------------------------------ f2: minimax semiring
@pytest.mark.parametrize("directed", [True, False])
def test_minimax_fw_equals_bruteforce(rng, directed):
    """Minimax FW == min over simple paths of the max edge (definition)."""
    for trial in range(25):
        n = int(rng.integers(2, 8))
        W = random_graph(rng, n, directed, float(rng.choice([0.4, 1.0])), lo=0, hi=9)
        assert np.array_equal(oracle.fw_minimax(W), oracle.brute_minimax_apsp(W)), (trial, W)


def test_minimax_equals_mst_path_max(rng):
    """Undirected minimax distance = the largest edge on the minimum spanning
    tree path (a classical property; MST by a plain Prim, independent of FW)."""
    n = 40
    W = random_graph(rng, n, False, 1.0, lo=1, hi=500)
    Wd = W.astype(np.int64)
    intree = np.zeros(n, bool)
    intree[0] = True
    adj = {i: [] for i in range(n)}
    best = Wd[0].copy()
    parent = np.zeros(n, int)
    for _ in range(n - 1):
        cand = np.where(intree, np.iinfo(np.int64).max, best)
        v = int(np.argmin(cand))
        intree[v] = True
        adj[v].append((parent[v], Wd[v, parent[v]]))
        adj[parent[v]].append((v, Wd[v, parent[v]]))
        upd = (~intree) & (Wd[v] < best)
        best[upd] = Wd[v][upd]
        parent[upd] = v
    exp = np.zeros((n, n), np.int64)
    for s in range(n):
        stack = [(s, 0)]
        seen = {s}
        while stack:
            x, mx = stack.pop()
            exp[s, x] = mx
            for y, w in adj[x]:
                if y not in seen:
                    seen.add(y)
                    stack.append((y, max(mx, w)))
    assert np.array_equal(oracle.fw_minimax(W), exp.astype(np.int32))


def test_minimax_need_update_is_safe(rng):
    """Theorem 4 carries over to minimax: unlisted pairs keep their distance."""
    for trial in range(40):
        n = int(rng.integers(3, 11))
        W = random_graph(rng, n, True, 1.0, lo=0, hi=7)
        D = oracle.fw_minimax(W)
        k = int(rng.integers(n))
        m = oracle.need_update_removal_minimax(D, k)
        W2, keep = _remove_from(W, k)
        D2 = oracle.fw_minimax(W2)
        Dk = D[np.ix_(keep, keep)]
        mk = m[np.ix_(keep, keep)]
        assert np.array_equal(D2[~mk], Dk[~mk])
        assert np.all(D2 >= Dk)


# ------------------------------------------- pins added in round 2
def _py_brute(W, combine):
    """Independent pure-Python enumeration of every simple path (n <= 6): the
    definition of the APSP matrix with the path cost folded by
    `combine` (sum: shortest path; max: minimax).  Floats in fp64."""
    W = np.asarray(W, np.float64)
    n = W.shape[0]
    out = np.full((n, n), np.inf)
    for s in range(n):
        out[s, s] = 0.0
        for t in range(n):
            if t == s:
                continue
            others = [v for v in range(n) if v not in (s, t)]
            for r in range(len(others) + 1):
                for mid in itertools.permutations(others, r):
                    p = [s, *mid, t]
                    c = 0.0
                    for a, b in zip(p[:-1], p[1:]):
                        c = combine(c, W[a, b])
                    out[s, t] = min(out[s, t], c)
    return out


def _float_graph(rng, n, directed):
    W = random_graph(rng, n, directed, 0.6, hi=1, dtype=np.float32)
    z = rng.random((n, n)) < 0.15           # some zero-weight edges
    if not directed:
        z = np.triu(z, 1)
        z = z | z.T
    W = np.where(z & np.isfinite(W), np.float32(0), W).astype(np.float32)
    np.fill_diagonal(W, 0)
    return W


@pytest.mark.parametrize("directed", [True, False])
def test_dijkstra_f64_rows_and_pair_equal_python_bruteforce(rng, directed):
    """oracle_dijkstra_rows_f64 / oracle_dijkstra_f64 (the fp32 full-size
    checkers) against an independent enumeration of simple paths, float
    weights with zeros and absent edges (+inf)."""
    for trial in range(20):
        n = int(rng.integers(2, 7))
        W = _float_graph(rng, n, directed)
        B = _py_brute(W, lambda c, w: c + w)
        D = oracle.dijkstra_rows(W, range(n))
        assert np.array_equal(np.isinf(D), np.isinf(B))
        fin = np.isfinite(B)
        assert np.allclose(D[fin], B[fin], rtol=1e-12, atol=0)
        assert np.allclose(oracle.dijkstra_cols(W, range(n))[fin], B[fin], rtol=1e-12, atol=0)
        s, t = (int(x) for x in rng.choice(n, 2, replace=False))
        d, path = oracle.dijkstra_pair(W, s, t)
        if np.isinf(B[s, t]):
            assert np.isinf(d) and path == []
        else:
            assert abs(d - B[s, t]) <= 1e-12 * max(B[s, t], 1e-300)
            assert oracle.path_is_valid(W, path, s, t)
            assert abs(oracle.path_weight(W, path) - d) <= 1e-12 * max(d, 1e-300)


@pytest.mark.parametrize("directed", [True, False])
def test_fw_minimax_f64_equals_python_bruteforce(rng, directed):
    """oracle_fw_minimax_f64 against the independent enumeration with the
    path cost = its largest edge; exact (max/min need no rounding)."""
    for trial in range(20):
        n = int(rng.integers(2, 7))
        W = _float_graph(rng, n, directed)
        assert np.array_equal(oracle.fw_minimax(W), _py_brute(W, max))


def _arc_crosses(n, i, j, a):
    """On the directed unit cycle the i -> j path is i, i+1, ..., j: it uses
    edge a -> a+1 iff a lies in [i, j) cyclically."""
    return (a - i) % n < (j - i) % n


def test_need_update_increase_exact_on_cycle():
    """Exact set (not only safety): on the directed unit cycle every pair has a
    unique shortest path, so raising edge u -> u+1 lists exactly the pairs
    whose arc crosses it (SURVEY §8(c-4) a4 closed form)."""
    n = 23
    D = oracle.fw(cycle(n))
    for u in (0, 7, n - 1):
        v = (u + 1) % n
        m = oracle.need_update_increase(D, u, v, 1, directed=True)
        exp = np.array([[i != j and _arc_crosses(n, i, j, u) for j in range(n)] for i in range(n)])
        assert np.array_equal(m, exp)


def test_need_update_increase_exact_on_undirected_path():
    """Undirected unit path: edge {u, u+1} lies on the unique i - j path iff
    min(i, j) <= u < max(i, j); both orientations are tested (DESIGN Q10)."""
    n = 19
    W = np.full((n, n), INF, np.int32)
    np.fill_diagonal(W, 0)
    a = np.arange(n - 1)
    W[a, a + 1] = 1
    W[a + 1, a] = 1
    D = oracle.fw(W)
    for u in (0, 5, n - 2):
        m = oracle.need_update_increase(D, u, u + 1, 1, directed=False)
        i, j = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
        exp = (np.minimum(i, j) <= u) & (u < np.maximum(i, j))
        assert np.array_equal(m, exp)


def test_need_update_removal_exact_on_cycle():
    """Removing k from the directed unit cycle lists exactly the pairs i, j != k
    whose arc passes through k as an interior node (Corollary 3, unique paths)."""
    n = 21
    D = oracle.fw(cycle(n))
    for k in (0, 9, n - 1):
        m = oracle.need_update_removal(D, k)
        exp = np.array([[i != j and i != k and j != k and (k - i) % n < (j - i) % n for j in range(n)]
                        for i in range(n)])
        assert np.array_equal(m, exp)
        assert oracle.cost(m, n)[0] == n - 2     # every other source loses some target


def test_need_update_removal_minimax_exact_on_increasing_path():
    """Minimax predicate, exact set: undirected path whose edge weights grow
    along it (w(a, a+1) = a + 1), so D[i][j] = max(i, j) off the diagonal.
    Removing k lists (i, j), both != k, iff max(D[i][k], D[k][j]) =
    max(i, j, k) equals max(i, j), i.e. iff max(i, j) > k: pairs straddling k
    and pairs beyond it (a detour through k costs no more than their own
    bottleneck edge — the ties the minimax algebra makes frequent, SURVEY
    f2); pairs below k are not listed (the detour's edge k is heavier)."""
    n = 15
    W = np.full((n, n), INF, np.int32)
    np.fill_diagonal(W, 0)
    a = np.arange(n - 1)
    W[a, a + 1] = a + 1
    W[a + 1, a] = a + 1
    D = oracle.fw_minimax(W)
    i, j = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    assert np.array_equal(D, np.where(i == j, 0, np.maximum(i, j)).astype(np.int32))
    for k in (1, 7, n - 2):
        m = oracle.need_update_removal_minimax(D, k)
        exp = (np.maximum(i, j) > k) & (i != j) & (i != k) & (j != k)
        assert np.array_equal(m, exp)
