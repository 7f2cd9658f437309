"""Probe: time single removals / adds at BJ.c4's size from one cold start.

    python scripts/update_probe.py [n] [reps]

Cold FW once, then `reps` removals of seeded random nodes and `reps` adds
(BJ.c4 edge distribution), each timed with CUDA events on the handle's
stream, plus the library's per-kernel-class profile of the removals.  Used
under ncu to capture the removal kernels of one update.
"""
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2412_15122_b200 as P  # noqa: E402
from paper_2412_15122_b200 import _lib as L  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
spec = synth.GraphSpec(n=n, directed=True, dtype="i32", kind=0, lo=1, hi=1000)
W = synth.graph(spec)
h = P.WarmAPSP(torch.from_numpy(W), directed=True, cap=n + reps + 1)
torch.cuda.synchronize()


def timed(fn):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(h.stream)
    out = fn()
    b.record(h.stream)
    torch.cuda.synchronize()
    return a.elapsed_time(b), out


L.apsp_profile_enable(h.h, True)
L.apsp_profile_reset(h.h)
rm = []
for r in range(reps):
    k = synth.uniform_int(1, 5, 100 + r, 0, 0, h.n - 1)
    ms, (_, info) = timed(lambda: h.remove_node(k))
    rm.append((ms, info.affected_pairs, info.affected_rows, info.rounds, info.path))
prof = {k: (round(v[0], 3), v[1]) for k, v in L.apsp_profile_read(h.h).items() if v[1]}
L.apsp_profile_reset(h.h)
ad = []
for r in range(reps):
    o, i = synth.node_edges(spec, 200 + r, h.n)
    od, idv = torch.from_numpy(o).cuda(), torch.from_numpy(i).cuda()
    torch.cuda.synchronize()
    ms, _ = timed(lambda: h.add_node(od, idv))
    ad.append(ms)
prof_add = {k: (round(v[0], 3), v[1]) for k, v in L.apsp_profile_read(h.h).items() if v[1]}
print(json.dumps({"n": n, "mirror_width": h.mirror_width, "remove_ms": [round(x[0], 4) for x in rm],
                  "remove_stats": [x[1:] for x in rm], "remove_profile_ms": prof,
                  "add_ms": [round(x, 4) for x in ad], "add_profile_ms": prof_add}))
