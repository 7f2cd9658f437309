import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..")); sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
import numpy as np, torch, oracle, synth
from conftest import random_graph
import paper_2412_15122_b200 as P
INF = synth.INF_I32
rng = np.random.default_rng(12345)
n = 200
W = random_graph(rng, n, True, 0.9, lo=1, hi=80)
a = P.WarmAPSP(torch.from_numpy(W), directed=True)
for trial in range(8):
    u, v = (int(x) for x in rng.choice(n, 2, replace=False))
    if trial == 3: u, v = n - 1, 0
    w_old = int(W[u, v]); w_new = int(rng.choice([max(0, w_old // 3), w_old * 5, INF, w_old + 1]))
    removed, info = a.modify_edge_readd(u, v, w_new)
    W[u, v] = w_new
    # full WT check
    bad = [(i, j, a.weight(i, j), W[i, j]) for i in range(n) for j in range(n) if (i * 7 + j) % 13 == 0 and a.weight(i, j) != W[i, j]]
    torch.cuda.synchronize()
    Dbad = int((a.D.cpu().numpy() != oracle.fw(W)).sum())
    print(trial, u, v, w_old, w_new, "removed", removed, info.kind, "n", a.n, "WT mismatches(sampled)", len(bad), bad[:4], "D mismatches", Dbad, flush=True)
