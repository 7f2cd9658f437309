"""Row-sharded protocol on CPU: world_size 2 over gloo (no GPU).

The library shards D by rows (apsp_layout) and exchanges, per SURVEY §8(e):
  * cold FW: the owner of pivot block K closes D_KK, computes the row panel
    D[K][:] and broadcasts it; every rank updates its column panel and the
    rest of its rows;
  * add node: every rank reduces its rows to a partial new row, all-reduce(min);
    the new column is local; rank-1 update on local rows;
  * remove node: the owner of row k broadcasts it; every rank detects and
    recomputes its own rows (no exchange); counters are all-reduced; the owner
    of row n-1 sends it to the owner of row k (swap-with-last).
This test replays exactly that decomposition with numpy compute per rank and
torch.distributed/gloo collectives, using the library's own host partition
function (apsp_layout), and requires the gathered D to equal the oracle's
cold APSP bit for bit (int32).  It checks the exchange schedule and the
decomposition's algebra; the kernels themselves are covered by -m gpu tests.
"""
import os
import socket

import numpy as np
import pytest

import oracle
import synth
from conftest import random_graph

torch = pytest.importorskip("torch")
dist = pytest.importorskip("torch.distributed")

INF = np.int64(synth.INF_I32)
TB = 128


def minplus(A, B):
    """C[i][j] = min_k A[i][k] + B[k][j] (int64, INF-saturated)."""
    C = np.full((A.shape[0], B.shape[1]), INF, np.int64)
    for k in range(A.shape[1]):
        C = np.minimum(C, A[:, k][:, None] + B[k, :][None, :])
    return np.minimum(C, INF)


def closure(T):
    T = T.copy()
    for k in range(T.shape[0]):
        T = np.minimum(T, T[:, k][:, None] + T[k, :][None, :])
    return T


def bcast(x, src):
    t = torch.from_numpy(np.ascontiguousarray(x))
    dist.broadcast(t, src=src)
    return t.numpy()


def gather_rows(Dl, row0, rows, n, world):
    parts = [None] * world
    dist.all_gather_object(parts, (row0, Dl[:max(0, min(rows, n - row0))].copy()))
    out = np.zeros((n, n), np.int64)
    for r0, blk in parts:
        if len(blk):
            out[r0:r0 + len(blk)] = blk[:, :n]
    return out


def worker(rank, world, port, W, cap, adds, removes, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2412_15122_b200 import _lib as L

        ld, row0, rows = L.apsp_layout(cap, world, rank)
        R = L.apsp_layout(cap, world, 0)[2]
        owner = lambda g: g // R
        n = W.shape[0]
        Wo = oracle.to_oracle(W)
        Wo[Wo >= oracle.INF64] = INF
        Wfull = np.full((cap, cap), INF, np.int64)
        Wfull[:n, :n] = Wo
        np.fill_diagonal(Wfull, 0)
        # ---- cold FW, blocked, row-sharded
        Dl = Wfull[row0:row0 + rows, :].copy()
        for K0 in range(0, n, TB):
            kb = min(TB, n - K0)
            o = owner(K0)
            if rank == o:
                lk = K0 - row0
                P = Dl[lk:lk + kb, :n].copy()
                P[:, K0:K0 + kb] = closure(P[:, K0:K0 + kb])
                Dkk = P[:, K0:K0 + kb]
                P = np.minimum(P, minplus(Dkk, P))
            else:
                P = np.zeros((kb, n), np.int64)
            P = bcast(P, o)
            Dkk = P[:, K0:K0 + kb]
            m = max(0, min(rows, n - row0))
            loc = Dl[:m, :n]
            loc[:, K0:K0 + kb] = np.minimum(loc[:, K0:K0 + kb], minplus(loc[:, K0:K0 + kb], Dkk))
            Dl[:m, :n] = np.minimum(loc, minplus(loc[:, K0:K0 + kb], P))
        D = gather_rows(Dl, row0, rows, n, world)
        ok_fw = np.array_equal(np.minimum(D, INF), oracle.to_oracle(oracle.fw(W)).clip(max=INF))
        # ---- add node(s): partial new row, all-reduce(min), rank-1 on local rows
        for (out_w, in_w) in adds:
            x = n
            m = max(0, min(rows, n - row0))
            loc = Dl[:m, :n]
            col = (loc + in_w[None, :n]).min(axis=1) if m else np.zeros(0, np.int64)
            part = (out_w[row0:row0 + m][:, None] + loc).min(axis=0) if m else np.full(n, INF)
            t = torch.from_numpy(np.minimum(part, INF).astype(np.int64))
            dist.all_reduce(t, op=dist.ReduceOp.MIN)
            row = np.minimum(t.numpy(), out_w[:n])
            Dl[:m, :n] = np.minimum(loc, col[:, None] + row[None, :])
            Dl[:m, x] = col
            if row0 <= x < row0 + rows:
                Dl[x - row0, :n] = row
                Dl[x - row0, x] = 0
            Wfull[x, :n] = out_w[:n]
            Wfull[:n, x] = in_w[:n]
            n += 1
        # ---- remove node(s): broadcast row k, local detection + local recompute,
        # counters all-reduced, swap-with-last by send/recv when owners differ
        for k in removes:
            m = max(0, min(rows, n - row0))
            rk = bcast(Dl[k - row0, :n] if owner(k) == rank else np.zeros(n, np.int64), owner(k))
            loc = Dl[:m, :n]
            lhs = loc[:, k][:, None] + rk[None, :]
            flag = (lhs == loc) & (loc < INF)
            flag[:, k] = False
            for li in range(m):
                flag[li, row0 + li] = False
            if row0 <= k < row0 + rows:
                flag[k - row0, :] = False
            cnt = torch.tensor([int(flag.sum())], dtype=torch.int64)
            dist.all_reduce(cnt)
            Wk = Wfull[:n, :n].copy()
            Wk[k, :] = INF
            Wk[:, k] = INF
            Wk[k, k] = 0
            loc = np.where(flag, Wk[row0:row0 + m, :n], loc)   # D0
            loc[:, k] = INF
            if row0 <= k < row0 + rows:
                loc[k - row0, :] = INF
                loc[k - row0, k] = 0
            for _ in range(n):   # Bellman rounds restricted to flagged pairs (a6 algebra)
                est = np.minimum(INF, (loc[:, :, None] + Wk[None, :, :]).min(axis=1))
                new = np.where(flag, np.minimum(loc, est), loc)
                if np.array_equal(new, loc):
                    break
                loc = new
            Dl[:m, :n] = loc
            last = n - 1
            if k != last:
                ok_, ol = owner(k), owner(last)
                if ok_ == ol == rank:
                    Dl[k - row0, :n] = Dl[last - row0, :n]
                elif rank == ol:
                    dist.send(torch.from_numpy(Dl[last - row0, :n].copy()), dst=ok_)
                elif rank == ok_:
                    buf = torch.zeros(n, dtype=torch.int64)
                    dist.recv(buf, src=ol)
                    Dl[k - row0, :n] = buf.numpy()
                m2 = max(0, min(rows, last - row0))
                Dl[:m2, k] = Dl[:m2, last]
                Wfull[k, :] = Wfull[last, :]
                Wfull[:, k] = Wfull[:, last]
                Wfull[k, k] = 0
            Wfull[last, :] = INF
            Wfull[:, last] = INF
            n -= 1
        D = gather_rows(Dl, row0, rows, n, world)
        # ---- sharded queries (f3, gather-free): row s of each query to every
        # rank (the owner writes it, the others zeros, all-reduce(sum)); every
        # rank tests the candidates k among ITS rows (D[s][k] from the shared
        # row, D[k][t] local); the hit lists are all-gathered; every rank then
        # solves (predecessor walk on the replicated W) — identical answers,
        # no exchange of outputs
        qs, qt = synth.query_pairs(3, n, 24)
        m = max(0, min(rows, n - row0))
        rowbuf = np.zeros((len(qs), n), np.int64)
        for b, s_ in enumerate(qs):
            if owner(s_) == rank:
                rowbuf[b] = Dl[s_ - row0, :n]
        rb = torch.from_numpy(rowbuf)
        dist.all_reduce(rb)
        rowbuf = rb.numpy()
        HCAP = n
        hits = np.zeros((len(qs), HCAP + 1), np.int64)    # count, then ids
        for b, (s_, t_) in enumerate(zip(qs, qt)):
            drow = rowbuf[b]
            st = drow[t_]
            if s_ == t_ or st >= INF:
                continue
            loc = [row0 + l for l in range(m)
                   if drow[row0 + l] < INF and Dl[l, t_] < INF and drow[row0 + l] + Dl[l, t_] == st]
            hits[b, 0] = len(loc)
            hits[b, 1:1 + len(loc)] = loc
        parts = [torch.zeros_like(torch.from_numpy(hits)) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(hits))
        PCAP = 64
        out = np.zeros((len(qs), 2 + PCAP), np.int64)      # dist, |C|, path (+1 so 0 = empty)
        Wq = np.minimum(Wfull[:n, :n], INF)
        for b, (s_, t_) in enumerate(zip(qs, qt)):
            drow = rowbuf[b]
            dst = drow[t_]
            cand = [int(x) for pt in parts for x in pt.numpy()[b, 1:1 + int(pt.numpy()[b, 0])]]
            path, cur = [t_], t_
            while cur != s_:   # predecessor walk: first m in (D[s][m], m) order with an exact last hop
                ok = [c for c in cand if (drow[c], c) < (drow[cur], cur) and Wq[c, cur] < INF
                      and drow[c] + Wq[c, cur] == drow[cur]]
                cur = min(ok, key=lambda c: (drow[c], c))
                path.append(cur)
            path = path[::-1]
            out[b, 0], out[b, 1] = dst, len(cand)
            out[b, 2:2 + len(path)] = np.array(path) + 1
        q.put((rank, ok_fw, D, int(cnt.item()) if removes else 0, (qs, qt, out)))
    finally:
        dist.destroy_process_group()


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("n,cap", [(300, 310), (257, 260)])
def test_row_sharded_protocol_world2(n, cap):
    import torch.multiprocessing as mp

    rng = np.random.default_rng(7)
    W = random_graph(rng, n, True, 0.8, lo=1, hi=60)
    adds = []
    hg = synth.HostGraph(W, True, cap=cap)
    for a in range(2):
        nn = hg.n
        o = np.full(cap, INF, np.int64)
        i = np.full(cap, INF, np.int64)
        o[:nn] = rng.integers(1, 60, nn)
        i[:nn] = rng.integers(1, 60, nn)
        adds.append((o, i))
        hg.add_node(o[:nn].astype(np.int32), i[:nn].astype(np.int32))
    removes = [5, hg.n - 1 - 1, 140]
    for k in removes:
        hg.remove_node(k)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, 2, port, W, cap, adds, removes, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    exp = oracle.to_oracle(oracle.fw(hg.W)).clip(max=INF)
    Wf = hg.W
    for rank, ok_fw, D, cnt, (qs, qt, out) in res:
        assert ok_fw, f"rank {rank}: sharded cold FW != oracle"
        assert np.array_equal(np.minimum(D, INF), exp), f"rank {rank}: sharded updates != oracle"
        assert np.array_equal(out, res[0][4][2]), "ranks disagree on the sharded query outputs"
        for b, (s_, t_) in enumerate(zip(qs, qt)):
            assert out[b, 0] == exp[s_, t_]
            assert out[b, 1] == len(oracle.candidates(exp, s_, t_))
            path = [int(x) - 1 for x in out[b, 2:] if x > 0]
            assert oracle.path_is_valid(Wf, path, s_, t_) and oracle.path_weight(Wf, path) == exp[s_, t_]
