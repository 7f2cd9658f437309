"""Run one cold FW (a1) at size n on a BJ.c4-shaped graph (profiling target)."""
import sys, os, dataclasses
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch, synth
import paper_2412_15122_b200 as P
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
dt = sys.argv[2] if len(sys.argv) > 2 else "i32"
spec = dataclasses.replace(synth.C4 if dt == "i32" else synth.C2, n=n)
W = synth.graph(spec)
h = P.WarmAPSP(torch.from_numpy(W), directed=spec.directed, cold_start=False)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for rep in range(2):
    e0.record(); h.cold_fw(); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"n={n} {dt} cold FW {ms:.2f} ms  {n**3 / ms / 1e9:.3f} Trelax/s")
