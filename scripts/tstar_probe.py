import json, os, sys
sys.path.insert(0, os.getcwd())
import torch, numpy as np
import synth
import paper_2412_15122_b200 as P
n = 32768
spec = synth.GraphSpec(n=n, directed=True, dtype="i32", kind=0, lo=1, hi=1000)
W = synth.graph(spec)
h = P.WarmAPSP(torch.from_numpy(W), directed=True, cap=n + 8)
D = h.D_local[:n, :n]
res = []
for r in range(3):
    o, i = synth.node_edges(spec, 200 + r, n)
    o = torch.from_numpy(o).cuda().long(); iv = torch.from_numpy(i).cuda().long()
    omin, t0 = o.min(0)
    Rb = omin + D[t0].max()
    S = torch.nonzero(o <= Rb).flatten()
    V = o[S, None] + D[S].long()              # |S| x n
    rowv = V.min(0).values
    tie = V == rowv[None, :]                   # minimiser mask
    # smallest t
    first = S[tie.int().argmax(0)]
    # smallest out among minimisers, then smallest t
    key = torch.where(tie, o[S, None] * (n + 1) + S[:, None], torch.full_like(V, 1 << 60))
    pref = key.min(0).values % (n + 1)
    # largest out preference
    key2 = torch.where(tie, -o[S, None] * (n + 1) + S[:, None], torch.full_like(V, 1 << 60))
    pref2 = (key2.min(0).values % (n + 1))
    # greedy hitting set
    cov = tie.clone(); chosen = 0; left = torch.ones(n, dtype=torch.bool, device='cuda')
    while left.any():
        c = (cov & left[None, :]).sum(1); b = int(c.argmax()); chosen += 1; left &= ~cov[b]
    imin = int(iv.min())
    s1 = {d: int((iv <= imin + d).sum()) for d in (0, 1, 2, 3)}
    res.append({"S": len(S), "Tfirst": int(first.unique().numel()), "Tsmallout": int(pref.unique().numel()),
                "Tlargeout": int(pref2.unique().numel()), "greedy": chosen, "S1": s1, "omin": int(omin), "Rb": int(Rb)})
print(json.dumps(res))
