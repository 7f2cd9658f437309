"""Probe: batched warm single-pair queries (a8) at one size, two leading dimensions.

    python scripts/query_probe.py [n] [pad]   # pad: extra capacity (changes ld)

Cold FW on a BJ.c4-distribution graph, then 1024 random queries through
sp_pair_query_batch, CUDA-event timed on the handle's stream.
"""
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2412_15122_b200 as P  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
pads = [int(x) for x in sys.argv[2:]] or [0]
spec = synth.GraphSpec(n=n, directed=True, dtype="i32", kind=0, lo=1, hi=1000)
W = synth.graph(spec)
for pad in pads:
    h = P.WarmAPSP(torch.from_numpy(W), directed=True, cap=n + pad)
    s, t = synth.query_pairs(1, n, 1024)
    sd, td = torch.from_numpy(s).cuda(), torch.from_numpy(t).cuda()
    for _ in range(3):
        h.query_batch(sd, td, path_cap=16)
    torch.cuda.synchronize()
    ms = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(h.stream)
        out = h.query_batch(sd, td, path_cap=16)
        b.record(h.stream)
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    ms.sort()
    print(json.dumps({"n": n, "ld": h.ld, "q": 1024, "ms_median": ms[2], "ms_min": ms[0],
                      "mean_candidates": out[3].float().mean().item(),
                      "bad": int((out[2] < 1).sum().item())}), flush=True)
    del h
    torch.cuda.empty_cache()
