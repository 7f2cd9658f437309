"""Diagnostic: for removals on a BJ.c4-shaped graph, how many flagged pairs
(need_update_list, ties included) actually change value, and where the time goes."""
import sys, os, dataclasses, json
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np, torch, synth
import paper_2412_15122_b200 as P
from paper_2412_15122_b200 import _lib as L
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
spec = dataclasses.replace(synth.C4, n=n)
W = synth.graph(spec)
h = P.WarmAPSP(torch.from_numpy(W), directed=True, cap=n + 8)
torch.cuda.synchronize()
rng = np.random.default_rng(0)
out = []
for trial in range(6):
    m = h.n
    k = int(rng.integers(m))
    Db = h.D.clone()
    L.apsp_profile_reset(h.h); L.apsp_profile_enable(h.h, True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); mf, info = h.remove_node(k); e1.record(); torch.cuda.synchronize()
    prof = L.apsp_profile_read(h.h); L.apsp_profile_enable(h.h, False)
    # relabel the old matrix: drop k, move last into k
    idx = list(range(m)); last = m - 1
    if k != last: idx[k] = last
    idx = idx[: m - 1]
    it = torch.tensor(idx, device=Db.device)
    Dold = Db.index_select(0, it).index_select(1, it)
    Dn = h.D
    changed = int((Dn != Dold).sum())
    rec = dict(k=k, ms=e0.elapsed_time(e1), affected=info.affected_pairs, rows=info.affected_rows,
               maxrow=info.max_row_affected, rounds=info.rounds, path=info.path, changed=changed,
               prof={c: round(v[0], 3) for c, v in prof.items() if v[1]})
    print(json.dumps(rec), flush=True)
    del Db, Dold
