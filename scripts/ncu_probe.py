"""One update of every kind at BJ.c4's size, for ncu captures of the hot kernels.

    python scripts/ncu_probe.py [n] [--no-mirror] [--fp32]

--no-mirror: APSP_OPT_MIRROR = 0 (the O(n^2) streams read the int32 D, 4 B
per entry); --fp32: the same kinds of updates on an fp32 graph of BJ.c2's
kind (complete, weights (m+1) 2^-24) at size n.

Cold FW (a1), one removal (a5 + a6), one add (a2), one tight-edge increase
(a4 + a6), one decrease (a3) and 1024 queries (a8), in that order.  Prints the
per-call CUDA-event times (meaningless under ncu; the plain run is the check
that the command exits 0 before profiling).
"""
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2412_15122_b200 as P  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
n = int(args[0]) if args else 32768
fp32 = "--fp32" in sys.argv
spec = (synth.GraphSpec(n=n, directed=True, dtype="f32", kind=2) if fp32 else
        synth.GraphSpec(n=n, directed=True, dtype="i32", kind=0, lo=1, hi=1000))
W = synth.graph(spec)
h = P.WarmAPSP(torch.from_numpy(W), directed=True, cap=n + 4, cold_start=False)
if "--no-mirror" in sys.argv:
    h.set_option(P._lib.OPT_MIRROR, 0)


def timed(fn):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(h.stream)
    out = fn()
    b.record(h.stream)
    torch.cuda.synchronize()
    return round(a.elapsed_time(b), 4), out


res = {}
res["cold_fw_ms"], _ = timed(h.cold_fw)
k = synth.uniform_int(1, 5, 7, 0, 0, n - 1)
res["remove_ms"], _ = timed(lambda: h.remove_node(k))
o, i = synth.node_edges(spec, 9, h.n)
od, idv = torch.from_numpy(o).cuda(), torch.from_numpy(i).cuda()
res["add_ms"], _ = timed(lambda: h.add_node(od, idv))
u = 123
row = W[u].astype(np.float64)
row[u] = np.inf
v = int(np.argmin(row))          # the cheapest out-edge of u: tight
res["increase_tight_ms"], info = timed(lambda: h.update_edge(u, v, W[u, v] * 10))
res["increase_pairs"] = info.affected_pairs
res["decrease_ms"], _ = timed(lambda: h.update_edge(u, v, W[u, v] / 2 if fp32 else 1))
s, t = synth.query_pairs(1, h.n, 1024)
sd, td = torch.from_numpy(s).cuda(), torch.from_numpy(t).cuda()
res["query1024_ms"], _ = timed(lambda: h.query_batch(sd, td, path_cap=16))
print(json.dumps(res))
