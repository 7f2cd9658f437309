"""Parity at BASELINE.json's full sizes (BJ.c2-c5), in the launch configuration
bench.py uses, on outputs the oracle can compute one by one: sampled rows and
columns by Dijkstra on the (mutated) host W, every query path validated, plus
properties that hold at any size (GPU warm == GPU cold FW, sparse == dense).
"""
import dataclasses

import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

INF = synth.INF_I32


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2412_15122_b200 as P
    return P


def rows_of(h, idx):
    torch.cuda.synchronize()
    it = torch.as_tensor(np.asarray(idx), device=h.D_local.device, dtype=torch.long)
    return h.D.index_select(0, it).cpu().numpy()


def cols_of(h, idx):
    torch.cuda.synchronize()
    it = torch.as_tensor(np.asarray(idx), device=h.D_local.device, dtype=torch.long)
    return h.D.index_select(1, it).cpu().numpy().T


def check_sampled_i32(h, W, rows, cols):
    exp_r = oracle.dijkstra_rows_i32(W, rows)
    exp_c = oracle.dijkstra_rows_i32(W, cols, reverse=True)
    assert np.array_equal(rows_of(h, rows), exp_r)
    assert np.array_equal(cols_of(h, cols), exp_c)


def check_sampled_f32(h, W, rows):
    exp = oracle.dijkstra_rows(W, rows)
    got = rows_of(h, rows).astype(np.float64)
    fin = np.isfinite(exp)
    assert np.array_equal(np.isfinite(got), fin)
    rel = np.abs(got[fin] - exp[fin]) / np.maximum(exp[fin], 1e-300)
    assert rel.max(initial=0) <= 1e-5


def test_bj_c2_fp32_updates_and_query(P):
    """BJ.c2: n=4096 undirected complete fp32 (0,1]; decrease x0.1, increase x10
    (random and tight variants); warm single-pair query."""
    spec = synth.C2
    W = synth.graph(spec)
    hg = synth.HostGraph(W, False)
    h = P.WarmAPSP(torch.from_numpy(W), directed=False)
    rng = np.random.default_rng(2)
    sample = rng.choice(spec.n, 24, replace=False)
    check_sampled_f32(h, hg.W, sample)
    torch.cuda.synchronize()
    for variant in ("random", "tight"):
        u, v = synth.random_edge(spec.seed, 100 if variant == "random" else 200, hg)
        if variant == "tight":
            d = float(rows_of(h, [u])[0, v])
            w_dec = np.float32(0.5 * d)
        else:
            w_dec = np.float32(hg.weight(u, v) * np.float32(0.1))
        h.update_edge(u, v, float(w_dec))
        hg.set_edge(u, v, w_dec)
        check_sampled_f32(h, hg.W, np.concatenate([[u, v], sample[:8]]))
        u2, v2 = synth.random_edge(spec.seed, 101 if variant == "random" else 201, hg)
        if variant == "tight":
            row = hg.W[u2].astype(np.float64)
            row[u2] = np.inf
            v2 = int(np.argmin(row))
        w_inc = np.float32(hg.weight(u2, v2) * np.float32(10))
        h.update_edge(u2, v2, float(w_inc))
        hg.set_edge(u2, v2, w_inc)
        check_sampled_f32(h, hg.W, np.concatenate([[u2, v2], sample[8:16]]))
    s, t = synth.query_pairs(spec.seed, spec.n, 4)
    D = None
    for q in range(4):
        d, path, nc = h.query(int(s[q]), int(t[q]))
        dd, _ = oracle.dijkstra_pair(hg.W, int(s[q]), int(t[q]))
        assert abs(d - dd) <= 1e-5 * dd
        assert oracle.path_is_valid(hg.W, path, int(s[q]), int(t[q]))
        assert abs(oracle.path_weight(hg.W, path) - dd) <= 1e-5 * dd


def test_bj_c3_remove_sparse_equals_dense(P):
    """BJ.c3: n=16384, density 0.9, U[1,1000]; remove one random node.  The
    sparse recompute and the dense FW fallback give bit-identical D, which
    matches the oracle on sampled rows/columns."""
    spec = synth.C3
    W = synth.graph(spec)
    k = synth.uniform_int(spec.seed, 5, 1, 0, 0, spec.n - 1)
    h = P.WarmAPSP(torch.from_numpy(W), directed=True)
    snap = h.D_local.clone()
    _, info_s = h.remove_node(k)
    Ds = h.D.clone()
    assert info_s.path == 2 and info_s.affected_pairs > 0
    # restart from the same state, force the dense path
    h2 = P.WarmAPSP(torch.from_numpy(W), directed=True, cold_start=False)
    h2.D_local.copy_(snap)
    del snap
    h2.set_option(0, 2)
    _, info_d = h2.remove_node(k)
    assert info_d.path == 3 and info_d.affected_pairs == info_s.affected_pairs
    assert torch.equal(Ds, h2.D)
    del h2
    hg = synth.HostGraph(W, True)
    hg.remove_node(k)
    rng = np.random.default_rng(3)
    rows = np.concatenate([[0, k], rng.choice(spec.n - 1, 14, replace=False)])
    check_sampled_i32(h, np.ascontiguousarray(hg.W), rows, rows[:8])


def _touched(up, n_before):
    """Node ids an update wrote (u, v, x and the moved slot)."""
    if up.kind == "add":
        return [n_before]                       # x
    if up.kind == "remove":
        return [up.k] if up.k < n_before - 1 else []   # slot k now holds node n-1
    return [up.u, up.v]


def check_sampled_i32_fast(h, hg, ids):
    """Rows and columns `ids` of the GPU D against oracle Dijkstra on the host
    graph (columns: Dijkstra on a transposed copy, a forward scan)."""
    n = hg.n
    Wv = hg.W
    exp_r = oracle.dijkstra_rows_i32(Wv, ids)
    WT = np.ascontiguousarray(Wv.T)
    exp_c = oracle.dijkstra_rows_i32(WT, ids)
    del WT
    assert np.array_equal(rows_of(h, ids), exp_r)
    assert np.array_equal(cols_of(h, ids), exp_c)
    assert exp_r.shape == (len(ids), n)


def test_bj_c4_sequence_64_updates_sampled_and_warm_equals_cold(P):
    """BJ.c4 in the bench's launch configuration (n=32768, the bench's cap and
    update sequence, seed 1): 64 updates (22 adds, 21 removals, 21 reweights),
    then 4 tight reweights (an increase of a cheapest out-edge x10, which runs
    detection + the sparse recompute, and a decrease to half the distance,
    which runs rank-1).  At t = 1, 8, 32, 64 and at the end: >= 64 rows and
    >= 64 columns — every id the recent updates touched (u, v, x, the moved
    slot) plus random ones — against oracle Dijkstra on the mutated host W
    (SURVEY §8(c-4)).  At the end GPU warm == GPU cold FW, bit-exact."""
    spec = synth.C4
    cap = spec.n + 64 + 4 * 23      # bench.py's cap (3 + 2*5 + 5 steps)
    W = synth.graph(spec)
    hg = synth.HostGraph(W, True, cap=cap)
    seq = synth.update_sequence(spec, synth.HostGraph(W, True, cap=cap), 0, 64)
    h = P.WarmAPSP(torch.from_numpy(W), directed=True, cap=cap)
    del W
    rng = np.random.default_rng(4)
    touched = []
    checks = {1, 8, 32, 64}
    for t, up in enumerate(seq, start=1):
        nb = hg.n
        if up.kind == "add":
            h.add_node(up.out_w, up.in_w)
            hg.add_node(up.out_w, up.in_w)
        elif up.kind == "remove":
            h.remove_node(up.k)
            hg.remove_node(up.k)
        else:
            h.update_edge(up.u, up.v, up.w_new)
            hg.set_edge(up.u, up.v, up.w_new)
        touched = [x for x in _touched(up, nb) if x < hg.n] + [x for x in touched if x < hg.n]
        if t in checks:
            ids = list(dict.fromkeys(touched))[:32]
            ids += [int(x) for x in rng.choice(hg.n, 64 - len(ids), replace=False) if int(x) not in ids]
            check_sampled_i32_fast(h, hg, np.asarray(ids, np.int64))
    # tight reweights: detection + sparse recompute, and rank-1
    Dn = None
    for q in range(2):
        u = int(rng.integers(hg.n))
        row = hg.W[u].astype(np.int64)
        row[u] = INF
        v = int(np.argmin(row))
        info = h.update_edge(u, v, int(hg.W[u, v]) * 10)
        assert info.kind == 2 and info.early_exit == 0 and info.path in (2, 3)
        hg.set_edge(u, v, int(hg.W[u, v]) * 10)
        u2, v2 = synth.random_edge(spec.seed, 1000 + q, hg)
        d = int(rows_of(h, [u2])[0, v2])
        w = max(0, d // 2)
        info = h.update_edge(u2, v2, w)
        assert info.kind == 1 and info.early_exit == 0 and info.path == 1
        hg.set_edge(u2, v2, w)
        touched = [u, v, u2, v2] + touched
    ids = list(dict.fromkeys(x for x in touched if x < hg.n))[:32]
    ids += [int(x) for x in rng.choice(hg.n, 64 - len(ids), replace=False) if int(x) not in ids]
    check_sampled_i32_fast(h, hg, np.asarray(ids, np.int64))
    Wn = np.ascontiguousarray(hg.W)
    warm = h.D.clone()
    del h
    torch.cuda.empty_cache()
    c = P.WarmAPSP(torch.from_numpy(Wn), directed=True)
    assert torch.equal(warm, c.D)


def test_bj_c5_fw_increase_and_1024_queries(P):
    """BJ.c5: n=65536 log-uniform [1,1e6]; cold FW, one edge increase x10
    (tight variant, so the recompute runs), 1024 warm queries: every path
    validated against W and the matrix; sampled rows vs the oracle."""
    spec = synth.C5
    W = synth.graph(spec)
    h = P.WarmAPSP(torch.from_numpy(W), directed=True)
    rng = np.random.default_rng(5)
    rows = rng.choice(spec.n, 4, replace=False)
    assert np.array_equal(rows_of(h, rows), oracle.dijkstra_rows_i32(W, rows))
    u = int(rows[0])
    row = W[u].astype(np.int64)
    row[u] = INF
    v = int(np.argmin(row))                       # cheapest out-edge: tight
    info = h.update_edge(u, v, int(W[u, v]) * 10)
    assert info.kind == 2 and info.early_exit == 0
    W[u, v] = W[u, v] * 10
    s, t = synth.query_pairs(spec.seed, spec.n, 1024)
    dist, paths, lens, nc = h.query_batch(s, t, path_cap=16)
    dist, paths, lens = dist.cpu().numpy(), paths.cpu().numpy(), lens.cpu().numpy()
    Dst = torch.stack([h.D[int(a), int(b)] for a, b in zip(s[:64], t[:64])]).cpu().numpy()
    assert np.array_equal(dist[:64], Dst)
    for q in range(1024):
        p = paths[q, : lens[q]].tolist()
        assert lens[q] > 0 and p[0] == s[q] and p[-1] == t[q] and len(set(p)) == len(p)
        assert sum(int(W[a, b]) for a, b in zip(p[:-1], p[1:])) == dist[q]
    chk = np.concatenate([[u], rows[1:3]])
    assert np.array_equal(rows_of(h, chk), oracle.dijkstra_rows_i32(W, chk))


def test_closed_form_cycle_at_65536(P):
    """Cold FW closed form at n=65536: directed unit cycle, D[i][j] = (j-i) mod n
    (hop counts up to n-1 stress every pivot-block dependency)."""
    n = 65536
    W = np.full((n, n), INF, np.int32)
    np.fill_diagonal(W, 0)
    W[np.arange(n), (np.arange(n) + 1) % n] = 1
    h = P.WarmAPSP(torch.from_numpy(W), directed=True)
    del W
    rng = np.random.default_rng(6)
    for i in rng.choice(n, 16, replace=False):
        got = rows_of(h, [int(i)])[0]
        assert np.array_equal(got, ((np.arange(n) - i) % n).astype(np.int32))
    # the query with the largest candidate set there is: C = all n nodes, the
    # path s = 0, 1, ..., n - 1 (no |C| cap)
    d, path, nc = h.query(0, n - 1, path_cap=n)
    assert d == n - 1 and nc == n and path == list(range(n))
