"""One tight-edge increase at BJ.c2 (n=4096 fp32 undirected) or BJ.c5
(n=65536 int32 log-uniform), after a warm-up one, inside the NVTX range
"probe" (ncu --nvtx --nvtx-include "probe/" lists just its launches).

    python scripts/update_probe.py c2|c5 [--bench-edge] [--heavy N]

--bench-edge: the tight increase scripts/bench_configs.py times (the cheapest
edge of synth.random_edge(seed, 2)'s tail), after one on the next node.
Prints each update's time, info and the heavy-row set it selected.
"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2412_15122_b200 as P  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
spec = synth.CONFIGS[cfg]
W = synth.graph(spec)
h = P.WarmAPSP(torch.from_numpy(W), directed=spec.directed)
if "--heavy" in sys.argv:   # APSP_OPT_HEAVY (0 default, -1 never, else the row threshold)
    h.set_option(P._lib.OPT_HEAVY, float(sys.argv[sys.argv.index("--heavy") + 1]))
INF = synth.INF_I32


def tight(u):
    row = W[u].astype(np.float64)
    row[u] = np.inf
    if W.dtype == np.int32:
        row[row >= INF] = np.inf
    return int(np.argmin(row))


us = (11, 12)
if len(sys.argv) > 2 and sys.argv[2] == "--bench-edge":   # bench_configs.py's tight increase
    u2, _ = synth.random_edge(spec.seed, 2, synth.HostGraph(W, spec.directed))
    us = ((u2 + 1) % spec.n, u2)
for it, u in enumerate(us):
    v = tight(u)
    w = W[u, v] * (10 if W.dtype == np.int32 else np.float32(10))
    if it == 1:
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_push("probe")
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    info = h.update_edge(u, v, float(w))
    b.record()
    torch.cuda.synchronize()
    if it == 1:
        torch.cuda.nvtx.range_pop()
    W[u, v] = w
    if not spec.directed:
        W[v, u] = w
    # the heavy-row set of this update (workspace layout: ..., heavy, small(64 KiB))
    ws = h.workspace
    ru = lambda x: (x + 255) // 256 * 256
    lcap = min(max(h.cap * h.cap // 32, 1 << 20), 1 << 28)
    ocap = max(lcap // 4, 1 << 18)
    off = ws.numel() - 65536 - ru(4 * ocap) - ru(512 + 4 * 32 * h.ld)   # [heavy | bigq | small]
    hs = ws[off:off + 36].view(torch.int32).cpu().tolist()
    print(cfg, it, round(a.elapsed_time(b), 4), info.as_dict(), "heavy", hs[0], hs[1:1 + min(hs[0], 8)])
