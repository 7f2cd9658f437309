"""Per-config measurements for BASELINE.json configs c1-c5 (besides bench.py's c4
sequence): device time of every hot-path call on its configured workload and
on the labelled tight-edge variants, CUDA events on the
handle's stream, median of R repeats from the same starting state.

    python scripts/bench_configs.py [c1 c2 c3 c5] > profiles/rNN_configs.jsonl
"""
import dataclasses
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2412_15122_b200 as P  # noqa: E402
from paper_2412_15122_b200 import _lib as L  # noqa: E402

INF = synth.INF_I32
_flush = None


def flush_l2():
    global _flush
    if _flush is None:
        _flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    _flush.fill_(1)


def timed(fn, flush=False):
    if flush:
        flush_l2()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    out = fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b), out


def emit(cfg, what, ms_list, n, extra=None):
    rec = {"config": cfg, "op": what, "n": n, "ms_median": statistics.median(ms_list),
           "ms_min": min(ms_list), "repeats": len(ms_list),
           "entries_per_s": n * n / (statistics.median(ms_list) / 1e3)}
    if extra:
        rec.update(extra)
    print(json.dumps(rec), flush=True)


def fresh(W, directed, D0, cap=None):
    h = P.WarmAPSP(torch.from_numpy(W), directed=directed, cap=cap, cold_start=False)
    h.D_local[: D0.shape[0], : D0.shape[1]].copy_(D0)
    h.sync_distances()   # warm start: not part of the timed update
    return h


def repeat_update(cfg, what, W, directed, D0, op, R=5, flush=False, cap=None):
    ms, info = [], None
    for _ in range(R):
        h = fresh(W, directed, D0, cap)
        t, info = timed(lambda: op(h), flush)
        ms.append(t)
        mw = h.mirror_width   # width of D's copy the streaming passes read (8 / 16; 0: D)
        del h
    d = info.as_dict() if hasattr(info, "as_dict") else {}
    emit(cfg, what, ms, W.shape[0], {"info": d, "l2_flushed": flush, "mirror_width": mw})


def cold(cfg, W, directed, R=3):
    h = P.WarmAPSP(torch.from_numpy(W), directed=directed, cold_start=False)
    ms = []
    for _ in range(R):
        t, _ = timed(h.cold_fw)
        ms.append(t)
    n = W.shape[0]
    emit(cfg, "cold_fw", ms, n, {"relax_per_s": n ** 3 / (statistics.median(ms) / 1e3)})
    D0 = h.D_local[:n, :n].clone()
    del h
    return D0


def tight_in(W, u):
    row = W[u].astype(np.float64)
    row[u] = np.inf
    row[row >= INF] = np.inf
    return int(np.argmin(row))


def c1():
    spec = synth.C1
    W = synth.graph(spec)
    D0 = cold("c1", W, True, R=5)
    o, i = synth.node_edges(spec, 0, spec.n)
    od, idv = torch.from_numpy(o).cuda(), torch.from_numpy(i).cuda()
    repeat_update("c1", "add_node", W, True, D0, lambda h: h.add_node(od, idv)[1], R=10, cap=spec.n + 1)


def c2():
    spec = synth.C2
    W = synth.graph(spec)
    D0 = cold("c2", W, False)
    hg = synth.HostGraph(W, False)
    u, v = synth.random_edge(spec.seed, 1, hg)
    w = float(np.float32(W[u, v]) * np.float32(0.1))
    for fl in (False, True):
        repeat_update("c2", "decrease_x0.1_random", W, False, D0, lambda h: h.update_edge(u, v, w), flush=fl)
    d = float(D0[u, v].item())
    repeat_update("c2", "decrease_tight_0.5D", W, False, D0, lambda h: h.update_edge(u, v, 0.5 * d), flush=True)
    u2, v2 = synth.random_edge(spec.seed, 2, hg)
    w2 = float(np.float32(W[u2, v2]) * np.float32(10))
    repeat_update("c2", "increase_x10_random", W, False, D0, lambda h: h.update_edge(u2, v2, w2), flush=True)
    v3 = tight_in(W, u2)
    w3 = float(np.float32(W[u2, v3]) * np.float32(10))
    repeat_update("c2", "increase_x10_tight", W, False, D0, lambda h: h.update_edge(u2, v3, w3), flush=True)
    s, t = synth.query_pairs(spec.seed, spec.n, 1)
    repeat_update("c2", "query", W, False, D0, lambda h: h.query(int(s[0]), int(t[0])), flush=True)


def c3():
    spec = synth.C3
    W = synth.graph(spec)
    D0 = cold("c3", W, True, R=2)
    k = synth.uniform_int(spec.seed, 5, 1, 0, 0, spec.n - 1)
    repeat_update("c3", "remove_node", W, True, D0, lambda h: h.remove_node(k)[1], R=3)

    def dense(h):
        h.set_option(0, 2)
        return h.remove_node(k)[1]
    repeat_update("c3", "remove_node_forced_dense", W, True, D0, dense, R=1)


def c5():
    spec = synth.C5
    W = synth.graph(spec)
    h = P.WarmAPSP(torch.from_numpy(W), directed=True, cold_start=False)
    t, _ = timed(h.cold_fw)
    n = spec.n
    emit("c5", "cold_fw", [t], n, {"relax_per_s": n ** 3 / (t / 1e3)})
    hg = synth.HostGraph.__new__(synth.HostGraph)   # no cap copy at 16 GiB: weights read from W
    u, v = synth.uniform_int(spec.seed, 5, 9, 1, 0, n - 1), synth.uniform_int(spec.seed, 5, 9, 2, 0, n - 2)
    v += v >= u
    ms = []
    t1, info = timed(lambda: h.update_edge(u, v, int(W[u, v]) * 10))
    emit("c5", "increase_x10_random", [t1], n, {"info": info.as_dict(), "mirror_width": h.mirror_width})
    vt = tight_in(W, u)
    u0 = (u + 1) % n   # an untimed tight increase first (the kernels' first launch loads them)
    v0 = tight_in(W, u0)
    h.update_edge(u0, v0, int(W[u0, v0]) * 10)
    W[u0, v0] = W[u0, v0] * 10
    t2, info = timed(lambda: h.update_edge(u, vt, int(W[u, vt]) * 10))
    emit("c5", "increase_x10_tight", [t2], n, {"info": info.as_dict(), "mirror_width": h.mirror_width})
    s, tt = synth.query_pairs(spec.seed, n, 1024)
    sd, td = torch.from_numpy(s).cuda(), torch.from_numpy(tt).cuda()
    for rep in range(3):
        t3, res = timed(lambda: h.query_batch(sd, td, path_cap=16))
        ms.append(t3)
    nc = res[3].float().mean().item()
    emit("c5", "query_batch_1024", ms, n, {"queries_per_s": 1024 / (statistics.median(ms) / 1e3),
                                           "mean_candidates": nc})
    t4, _ = timed(lambda: h.query(int(s[0]), int(tt[0])))
    emit("c5", "query_single", [t4], n)
    # a large batch (t-grouped: 16384 queries over 256 targets, f3)
    s2, t2q = synth.query_pairs(spec.seed + 1, n, 16384)
    t2q = t2q[np.arange(16384) % 256]   # 64 queries per target
    sd2, td2 = torch.from_numpy(s2).cuda(), torch.from_numpy(np.ascontiguousarray(t2q)).cuda()
    ms2 = []
    for rep in range(3):
        t5, res2 = timed(lambda: h.query_batch(sd2, td2, path_cap=16))
        ms2.append(t5)
    emit("c5", "query_batch_16384_grouped", ms2, n, {"queries_per_s": 16384 / (statistics.median(ms2) / 1e3),
                                                    "targets": 256,
                                                    "mean_candidates": res2[3].float().mean().item()})


def c4f1():
    """f1 ablation at BJ.c4's size: the paper's edge modification (remove the
    cheaper endpoint + re-add) vs the direct decrease/increase path,
    on the same random reweights (factor in [0.1, 10]) and on tight edges."""
    spec = synth.C4
    n = spec.n
    W = synth.graph(spec)
    h = P.WarmAPSP(torch.from_numpy(W), directed=True)
    D0 = h.D_local[:n, :n].clone()
    del h
    hg = synth.HostGraph.__new__(synth.HostGraph)
    hg.buf, hg.n, hg.inf, hg.directed, hg.dtype = W, n, INF, True, W.dtype
    edges = []
    for t in range(3):
        u, v = synth.random_edge(spec.seed, 1000 + t, hg)
        edges.append(("random", u, v, synth.new_weight(W[u, v], synth.reweight_factor(spec.seed, 1000 + t), W.dtype)))
    for t in range(2):
        u = 31 + 977 * t
        v = tight_in(W, u)
        edges.append(("tight_x10", u, v, int(W[u, v]) * 10))
    for kind, u, v, w in edges:
        repeat_update("c4", f"modify_readd_{kind}", W, True, D0, lambda h: h.modify_edge_readd(u, v, w)[1], R=2)
        repeat_update("c4", f"update_edge_{kind}", W, True, D0, lambda h: h.update_edge(u, v, w), R=2)


if __name__ == "__main__":
    which = sys.argv[1:] or ["c1", "c2", "c3", "c5", "c4f1"]
    for c in which:
        globals()[c]()
        torch.cuda.empty_cache()
