import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..")); sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
import numpy as np, torch, oracle
from conftest import random_graph
import paper_2412_15122_b200 as P
rng = np.random.default_rng(12345)
n = 260
for directed in (False,):
    W = random_graph(rng, n, directed, 1.0, lo=1, hi=100)
    h = P.WarmAPSP(torch.from_numpy(W), directed=directed)
    for trial in range(12):
        torch.cuda.synchronize(); D = h.D.cpu().numpy().astype(np.int64)
        assert np.array_equal(D, oracle.fw(W)), "pre"
        u, v = (int(x) for x in rng.choice(n, 2, replace=False))
        w_old = int(W[u, v])
        w_new = max(0, int(D[u, v]) // 2) if trial % 2 else max(0, w_old // 10)
        if w_new >= w_old: continue
        info = h.update_edge(u, v, w_new)
        W[u, v] = w_new
        if not directed: W[v, u] = w_new
        torch.cuda.synchronize(); G = h.D.cpu().numpy()
        R = np.minimum(D, D[:, u][:, None] + w_new + D[v, :][None, :])
        if not directed: R = np.minimum(R, D[:, v][:, None] + w_new + D[u, :][None, :])
        O = oracle.fw(W)
        bad = np.argwhere(G != O)
        print(directed, trial, u, v, w_old, w_new, D[u, v], info.as_dict()["early_exit"], "formula==oracle", np.array_equal(R, O), "bad", len(bad))
        for (i, j) in bad[:5]:
            print("   ", i, j, "gpu", G[i, j], "oracle", O[i, j], "D", D[i, j], "t1", D[i, u] + w_new + D[v, j], "t2", D[i, v] + w_new + D[u, j])
        if len(bad): sys.exit(1)
