"""Probe: BJ.c2 (n=4096 undirected fp32) tight-edge increase, per-kernel-class
profile and wall time, from one cold start (restored between repeats)."""
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2412_15122_b200 as P  # noqa: E402
from paper_2412_15122_b200 import _lib as L  # noqa: E402

spec = synth.C2
W = synth.graph(spec)
h = P.WarmAPSP(torch.from_numpy(W), directed=False)
D0 = h.D_local.clone()
hg = synth.HostGraph(W, False)
u2, _ = synth.random_edge(spec.seed, 2, hg)
row = W[u2].astype(np.float64)
row[u2] = np.inf
v3 = int(np.argmin(row))
w3 = float(np.float32(W[u2, v3]) * np.float32(10))
out = []
for rep in range(4):
    h.close()
    h = P.WarmAPSP(torch.from_numpy(W), directed=False, cold_start=False)
    h.D_local.copy_(D0)
    h.sync_distances()
    torch.cuda.synchronize()
    L.apsp_profile_enable(h.h, rep == 3)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(h.stream)
    info = h.update_edge(u2, v3, w3)
    b.record(h.stream)
    torch.cuda.synchronize()
    out.append(round(a.elapsed_time(b), 4))
prof = {k: (round(v[0], 4), v[1]) for k, v in L.apsp_profile_read(h.h).items() if v[1]}
print(json.dumps({"ms": out, "info": info.as_dict(), "profile_ms": prof}))
