"""One update of each kind on a BJ.c4-shaped graph (ncu / timing target).

    python scripts/one_update.py [n] [kinds...]    kinds: add remove dec inc
"""
import dataclasses
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2412_15122_b200 as P  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
kinds = sys.argv[2:] or ["add", "remove", "dec", "inc"]
spec = dataclasses.replace(synth.C4, n=n)
W = synth.graph(spec)
h = P.WarmAPSP(torch.from_numpy(W), directed=True, cap=n + 8)
torch.cuda.synchronize()
o, i = synth.node_edges(spec, 0, n)
od, idv = torch.from_numpy(o).cuda(), torch.from_numpy(i).cuda()
for kind in kinds:
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    if kind == "add":
        _, info = h.add_node(od[: h.n], idv[: h.n])
    elif kind == "remove":
        _, info = h.remove_node(12345 % h.n)
    elif kind == "dec":
        u, v = 7, 4242
        d = int(h.D[u, v].item())
        info = h.update_edge(u, v, max(1, d // 2))
    else:
        u = 99
        row = W[u].astype(np.int64)
        row[u] = 1 << 40
        v = int(np.argmin(row))
        info = h.update_edge(u, v, int(W[u, v]) * 10)
    b.record()
    torch.cuda.synchronize()
    print(kind, f"{a.elapsed_time(b):.3f} ms", info.as_dict(), flush=True)
