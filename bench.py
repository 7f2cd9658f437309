#!/usr/bin/env python
"""bench.py — warm-start APSP update throughput on B200 (BASELINE.json metric).

Metric (BJ.metric): "APSP entries updated/s per warm-start update; ms/update
at n=32768".  Workload: BJ.c4 — n=32768 directed complete graph, int32
weights U[1,1000], a seeded sequence of updates (1/3 add-node, 1/3
remove-node, 1/3 edge reweight by a log-uniform factor in [0.1, 10]; DESIGN.md
Q18).  One "step" = 64 consecutive updates of that sequence (every hot-path
row a2-a7 the sequence exercises); entries updated per update = n_after^2.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1: launched under torch.distributed.run, one rank per GPU; D is
row-sharded over the ranks (NCCL over NVLink inside the library), every
rank applies the same updates, time = max over ranks.

--impl reference: the CPU oracle (plain Floyd–Warshall, cold, as the paper's
comparator) timed on the host cores on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

UPDATES_PER_STEP = 64
METRIC = "APSP entries updated/s per warm-start update (BJ.c4 sequence)"
UNIT = "entries/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--n", type=int, default=synth.C4.n)
    p.add_argument("--seed", type=int, default=1)
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-cold", action="store_true", help="skip timing one cold FW")
    p.add_argument("--json-extra", default=None, help="write the detailed report here")
    p.add_argument("--no-verify", action="store_true", help="skip the post-run oracle check")
    p.add_argument("--no-int32", action="store_true",
                   help="skip the profiled pass on the int32 streams (APSP_OPT_MIRROR=0)")
    p.add_argument("--verify-samples", type=int, default=16)
    return p.parse_args()


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            mp = json.load(f)
        return mp, "measured"
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self):
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self, gpu_index=None):
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        with open(self.path) as f:
            for line in f:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    rows.append((int(parts[0]), float(parts[1]), float(parts[2]), parts[5:9]))
                except ValueError:
                    continue
        os.unlink(self.path)
        if gpu_index is not None:
            sel = [r for r in rows if r[0] == gpu_index]
            rows = sel or rows
        if not rows:
            return None
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i, v in enumerate(r[3]) if v.lower().startswith("active")})
        under = [r[1] for r in rows if r[1] > 400] or [r[1] for r in rows]
        return {"sm_mhz": statistics.median(under), "sm_max_mhz": max(r[2] for r in rows),
                "reasons": reasons, "samples": len(rows)}


# ----------------------------------------------------------------------------- oracle leg
def oracle_pivot_time(W: np.ndarray, budget_s: float = 12.0, max_pivots: int = 64):
    """Time the CPU oracle's Floyd–Warshall (cold recompute per update) on a
    bounded sample: `p` pivots of the full-size n x n int64 matrix.  Returns
    (seconds per pivot, pivots timed)."""
    import oracle

    A = oracle.to_oracle(W)
    n = A.shape[0]
    t0 = time.perf_counter()
    oracle.fw_raw_i64(A, 0, 1)
    t1 = time.perf_counter() - t0
    p = int(max(2, min(max_pivots, budget_s / max(t1, 1e-6))))
    t0 = time.perf_counter()
    oracle.fw_raw_i64(A, 1, 1 + p)
    tp = (time.perf_counter() - t0) / p
    del A
    return tp, p, n


def cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


def run_reference(args, rank, world):
    """--impl reference: the oracle (cold FW per update) on the host cores."""
    if rank != 0:
        return
    spec = dataclasses.replace(synth.C4, n=args.n, seed=args.seed)
    W = synth.graph(spec)
    n = spec.n
    step_times = []
    pivots = 0
    for s in range(args.warmup + args.steps):
        tp, p, _ = oracle_pivot_time(W, budget_s=4.0, max_pivots=16)
        if s >= args.warmup:
            # one step = 64 updates, each an oracle cold FW (n pivots) at n
            step_times.append(UPDATES_PER_STEP * n * tp)
            pivots += p
    step_s = statistics.median(step_times)
    value = UPDATES_PER_STEP * n * n / step_s
    c = cores()
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_s * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int64",
        "data": "synthetic (seeded BJ.c4 graph, U[1,1000])",
        "config": {"workload": "BJ.c4", "n": n, "updates_per_step": UPDATES_PER_STEP, "directed": True},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": c, "kind": "oracle",
                         "sample": f"{pivots} Floyd-Warshall pivots of the n={n} int64 matrix timed, "
                                   f"extrapolated x n per update (cold recompute), {UPDATES_PER_STEP} updates/step"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- post-run check
def final_check(h, hg, seq, rank, world, pg, dev, samples=16):
    """Sampled rows and columns of the final D (every update of the run applied)
    against oracle Dijkstra on the host graph: the ids the last updates touched
    (x, the moved slot, u, v) plus random ones.  Rows / column slices are
    gathered from their owners when D is sharded; rank 0 compares."""
    import torch

    n = h.n
    ids = []
    for up in reversed(seq):
        cand = {"add": [up.n_before], "remove": [up.k], "reweight": [up.u, up.v]}[up.kind]
        ids += [x for x in cand if 0 <= x < n and x not in ids]
        if len(ids) >= samples // 2:
            break
    rng = np.random.default_rng(7)
    for x in rng.permutation(n):
        if len(ids) >= samples:
            break
        if int(x) not in ids:
            ids.append(int(x))
    ids = np.asarray(ids[:samples], np.int64)
    torch.cuda.synchronize(dev)
    lo, hi = min(h.row0, n), min(h.row0 + h.rows, n)
    it = torch.as_tensor(ids, device=dev)
    cols_local = h.D.index_select(1, it).cpu().numpy()          # (hi - lo) x samples
    mine = [(int(i), h.D[int(i) - lo].cpu().numpy()) for i in ids if lo <= i < hi]
    if world > 1:
        got_c, got_r = [None] * world, [None] * world
        pg.all_gather_object(got_c, (lo, cols_local))
        pg.all_gather_object(got_r, mine)
    else:
        got_c, got_r = [(lo, cols_local)], [mine]
    if rank != 0:
        return None
    import oracle   # test infrastructure: the checker, never on the product path

    C = np.full((n, len(ids)), -1, np.int64)
    for l0, blk in got_c:
        C[l0:l0 + blk.shape[0]] = blk
    R = dict(x for part in got_r for x in part)
    Rm = np.stack([R[int(i)] for i in ids])
    t0 = time.perf_counter()
    Wv = hg.W
    exp_r = oracle.dijkstra_rows_i32(Wv, ids)
    WT = np.ascontiguousarray(Wv.T)
    exp_c = oracle.dijkstra_rows_i32(WT, ids).T
    del WT
    dt = time.perf_counter() - t0
    bad_r = int(np.count_nonzero(Rm != exp_r))
    bad_c = int(np.count_nonzero(C != exp_c))
    return {"ok": bad_r == 0 and bad_c == 0, "n": n, "updates_applied": len(seq), "rows": len(ids),
            "cols": len(ids), "ids": ids.tolist(), "mismatches": bad_r + bad_c,
            "oracle": "Dijkstra rows + columns (transposed W) on the host graph", "oracle_s": round(dt, 2)}


# ----------------------------------------------------------------------------- our leg
def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        if world > 1:
            import torch.distributed as dist  # noqa: F401
        run_reference(args, rank, world)
        return

    import torch

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    pg = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
        pg = dist

    import paper_2412_15122_b200 as P
    from paper_2412_15122_b200 import _lib as L

    spec = dataclasses.replace(synth.C4, n=args.n, seed=args.seed)
    n0 = spec.n
    # warm-up, timed, per-update-timing, e2e and profiled steps each consume their own updates
    steps_total = (args.warmup + 3 * args.steps + (0 if args.no_e2e else args.steps) +
                   (0 if args.no_int32 else args.steps))
    cap = n0 + UPDATES_PER_STEP + 4 * steps_total
    t_setup = time.perf_counter()
    W = synth.graph(spec)
    hg = synth.HostGraph(W, True, cap=cap)
    seq = synth.update_sequence(spec, hg, 0, steps_total * UPDATES_PER_STEP)
    # hg now holds W after every update the run applies: the post-run check
    # compares the GPU's final state with the oracle on it (rank 0 keeps it)
    hg_final = hg if rank == 0 else None
    del hg

    nccl_id = None
    if world > 1:
        obj = [L.apsp_nccl_unique_id() if rank == 0 else None]
        pg.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    stream = torch.cuda.current_stream(dev)
    h = P.WarmAPSP(torch.from_numpy(W), directed=True, cap=cap, device=dev, stream=stream, rank=rank,
                   world=world, nccl_id=nccl_id, cold_start=False)
    del W

    def barrier():
        if pg is not None:
            pg.barrier()
        torch.cuda.synchronize(dev)

    def max_over_ranks(x):
        if pg is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        return float(t.item())

    # cold start: D := APSP(W) by blocked FW (a1), timed once (warm-vs-cold speedup)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    h.cold_fw()
    e1.record(stream)
    barrier()
    cold_ms = max_over_ranks(e0.elapsed_time(e1))

    # device-resident add-node vectors for the device-timed steps
    dvecs = {}
    for up in seq:
        if up.kind == "add":
            dvecs[up.t] = (torch.from_numpy(up.out_w).to(dev), torch.from_numpy(up.in_w).to(dev))
    setup_s = time.perf_counter() - t_setup

    per_update = []   # (kind, ms, n_after, info): the per-update-timing pass
    timed_n = []      # n_after of every update of the timed region

    def run_step(s, mode="plain"):
        """One step's 64 updates through the C ABI.  mode "timed": nothing but
        the library calls (n_after kept for the metric); "events": CUDA events
        around every call (the per-type breakdown); "plain": the calls only."""
        events = mode == "events"
        ups = seq[s * UPDATES_PER_STEP:(s + 1) * UPDATES_PER_STEP]
        evs = []
        infos = []
        for up in ups:
            if events:
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record(stream)
            if up.kind == "add":
                o, i = dvecs[up.t]
                _, info = L.apsp_add_node(h.h, o.data_ptr(), i.data_ptr())
            elif up.kind == "remove":
                _, info = L.apsp_remove_node(h.h, up.k)
            else:
                info = L.apsp_update_edge(h.h, up.u, up.v, float(up.w_new))
            if events:
                b.record(stream)
                evs.append((a, b))
            infos.append((up.kind, info))
        if mode == "timed":
            timed_n.extend(info.n_after for _, info in infos)
        if events:
            torch.cuda.synchronize(dev)
            for (a, b), (kind, info) in zip(evs, infos):
                per_update.append((kind, a.elapsed_time(b), info.n_after, info.as_dict()))

    for s in range(args.warmup):
        run_step(s)
    torch.cuda.synchronize(dev)

    # ---------------- timed region (device-resident inputs)
    clk = ClockSampler()
    if rank == 0:
        clk.start()
    launches0 = h.launches()
    barrier()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    torch.cuda.nvtx.range_push("timed")   # (ncu --nvtx --nvtx-include "timed/": the timed region's launches)
    for s in range(args.warmup, args.warmup + args.steps):
        run_step(s, "timed")
    torch.cuda.nvtx.range_pop()
    # (the library's side stream may still hold the last removal's shortlist
    # upkeep, joined lazily by the next update: drain every stream first)
    torch.cuda.synchronize(dev)
    t1.record(stream)
    barrier()
    total_ms = max_over_ranks(t0.elapsed_time(t1))
    launches = h.launches() - launches0
    clocks = clk.stop(gpu_index=None) if rank == 0 else None


    entries = sum(na * na for na in timed_n)
    value = entries / (total_ms / 1e3)
    ms_per_step = total_ms / args.steps

    # ---------------- per-update times (CUDA events around every call): the
    # per-type breakdown, on the next K steps (not the timed region)
    s_pu = args.warmup + args.steps
    for s in range(s_pu, s_pu + args.steps):
        run_step(s, "events")

    # ---------------- e2e: public API with host buffers, copies inside the timed region
    e2e = None
    if not args.no_e2e:
        s_lo = args.warmup + 2 * args.steps
        pinned = {}
        for up in seq[s_lo * UPDATES_PER_STEP:]:
            if up.kind == "add":
                pinned[up.t] = (torch.from_numpy(up.out_w).pin_memory(), torch.from_numpy(up.in_w).pin_memory())
        res_host = torch.empty(cap, dtype=torch.int32).pin_memory()
        h2d = d2h = 0
        entries_e2e = 0
        barrier()
        q0 = torch.cuda.Event(enable_timing=True)
        q1 = torch.cuda.Event(enable_timing=True)
        q0.record(stream)
        for s in range(s_lo, s_lo + args.steps):
            ups = seq[s * UPDATES_PER_STEP:(s + 1) * UPDATES_PER_STEP]
            for up in ups:
                if up.kind == "add":
                    o, i = pinned[up.t]
                    od = o.to(dev, non_blocking=True)
                    idv = i.to(dev, non_blocking=True)
                    h2d += o.numel() * 4 * 2
                    x, info = h.add_node(od, idv)
                elif up.kind == "remove":
                    _, info = h.remove_node(up.k)
                else:
                    info = h.update_edge(up.u, up.v, up.w_new)
                entries_e2e += info.n_after * info.n_after
            # the step's result back to the host: row 0 of D (owner) — distances from node 0
            nn = h.n
            if h.row0 == 0:
                res_host[:nn].copy_(h.D_local[0, :nn], non_blocking=True)
                d2h += nn * 4
        torch.cuda.synchronize(dev)   # (every stream of the handle drained, as above)
        q1.record(stream)
        barrier()
        e2e_ms = max_over_ranks(q0.elapsed_time(q1))
        e2e = {"value": entries_e2e / (e2e_ms / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": h2d // args.steps, "d2h_bytes_per_step": d2h // args.steps,
               "ms_per_step": e2e_ms / args.steps}

    # ---------------- profiled pass (not the timed one): the library brackets
    # every kernel with CUDA events on its stream -> per-class time and work
    L.apsp_profile_reset(h.h)
    L.apsp_profile_enable(h.h, True)
    barrier()
    p0 = torch.cuda.Event(enable_timing=True)
    p1 = torch.cuda.Event(enable_timing=True)
    p0.record(stream)
    s_prof = args.warmup + 2 * args.steps + (0 if args.no_e2e else args.steps)
    for s in range(s_prof, s_prof + args.steps):
        run_step(s)
    torch.cuda.synchronize(dev)
    p1.record(stream)
    barrier()
    prof_total_ms = max_over_ranks(p0.elapsed_time(p1))
    L.apsp_profile_enable(h.h, False)
    prof = L.apsp_profile_read(h.h)

    # ---------------- profiled pass on the 4-byte streams: the same kind of
    # steps with the saturated mirror switched off (APSP_OPT_MIRROR = 0), so
    # detection, add-node pass 1 and rank-1 stream the int32 D itself at
    # SURVEY §8(d-4)'s 4 bytes per entry (after every timed number is taken)
    prof32 = None
    if not args.no_int32:
        L.apsp_set_option(h.h, L.OPT_MIRROR, 0)
        s32 = s_prof + args.steps
        run_step(s32)     # the first update after the switch drops the mirror
        torch.cuda.synchronize(dev)
        L.apsp_profile_reset(h.h)
        L.apsp_profile_enable(h.h, True)
        barrier()
        for s in range(s32 + 1, s32 + args.steps):
            run_step(s)
        barrier()
        L.apsp_profile_enable(h.h, False)
        prof32 = L.apsp_profile_read(h.h)

    # ---------------- K13: the roofline denominators measured on this device
    k13 = None
    try:
        buf = torch.empty(1 << 31, dtype=torch.uint8, device=dev)   # 2 GiB > L2
        sptr = stream.cuda_stream
        k13 = {"int32_relax_per_s": L.apsp_microbench(0, buf.data_ptr(), 4, sptr),
               "fp32_relax_per_s": L.apsp_microbench(1, buf.data_ptr(), 4, sptr),
               "int16x2_relax_per_s": L.apsp_microbench(2, buf.data_ptr(), 4, sptr),
               "hbm_read_gbs": L.apsp_microbench(3, buf.data_ptr(), buf.numel(), sptr) / 1e9,
               "hbm_rmw_gbs": L.apsp_microbench(4, buf.data_ptr(), buf.numel(), sptr) / 1e9}
        del buf
        torch.cuda.empty_cache()
    except Exception as e:   # measurement hook only: report, never fail the bench
        k13 = {"error": str(e)[:200]}

    # ---------------- roofline of the dominant kernel class
    mp, peak_kind = peaks()
    hbm_peak = float(mp.get("hbm_gbs", 6650.0))
    cls_ms = {k: v[0] for k, v in prof.items() if k != "other"}
    dom = max(cls_ms, key=cls_ms.get)
    ms_d, cnt_d, work_d = prof[dom]
    traffic = None
    traffic32 = {}
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            with open(tpath) as f:
                tj = json.load(f)
            traffic = tj.get(dom)
            traffic = traffic if isinstance(traffic, (int, float)) else None
            traffic32 = {k: v for k, v in (tj.get("int32") or {}).items() if isinstance(v, (int, float))}
        except Exception:
            traffic = None
    if dom.startswith("fw"):
        sm_mhz = float(mp.get("sm_max_mhz", 1965.0))
        peak = 148 * 64 * sm_mhz * 1e6 / 1e12     # VIADDMNMX: 64 relaxations/clk/SM
        if k13 and k13.get("int32_relax_per_s"):
            peak = k13["int32_relax_per_s"] / 1e12   # measured (K13)
        achieved = work_d / (ms_d / 1e3) / 1e12
        roof = {"bound": "alu", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "Trelax/s",
                "frac": achieved / peak, "traffic": traffic, "launches": cnt_d}
    else:
        achieved = work_d / (ms_d / 1e3) / 1e9 if ms_d > 0 else 0.0
        roof = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                "frac": achieved / hbm_peak, "traffic": traffic, "launches": cnt_d,
                "peak_kind": f"{peak_kind} copy bandwidth"}
        if k13 and k13.get("hbm_read_gbs"):   # the same kernel against the measured read-only stream
            roof["k13_read_gbs"] = k13["hbm_read_gbs"]
            roof["frac_of_k13_read"] = achieved / k13["hbm_read_gbs"]
    roof["basis"] = ("algorithmic bytes of the stream the kernel reads: the int8 mirror of D (1 B/entry) "
                     "while every distance is < 0x7F, else int16 (2 B) or D itself (4 B); DESIGN.md §6")
    roof32 = None
    if prof32 is not None:
        # the dominant O(n^2) stream class with the mirror off, on §8(d-4)'s 4 B/entry
        cand = {k: v for k, v in prof32.items() if k in ("detect", "add_pass1", "rank1") and v[0] > 0}
        if cand:
            d32 = max(cand, key=lambda k: cand[k][0])
            ms32, c32, w32 = prof32[d32]
            a32 = w32 / (ms32 / 1e3) / 1e9
            roof32 = {"bound": "hbm", "kernel": d32, "achieved": a32, "peak": hbm_peak, "unit": "GB/s",
                      "frac": a32 / hbm_peak, "traffic": traffic32.get(d32), "launches": c32,
                      "peak_kind": f"{peak_kind} copy bandwidth",
                      "basis": "int32 D, 4 B per entry read (SURVEY §8(d-4)); APSP_OPT_MIRROR = 0",
                      "classes": {k: {"ms": round(v[0], 3), "launches": v[1],
                                      "achieved_gbs": round(v[2] / (v[0] / 1e3) / 1e9, 1) if v[0] > 0 else None}
                                  for k, v in prof32.items() if v[1] > 0}}
            if k13 and k13.get("hbm_read_gbs"):
                roof32["frac_of_k13_read"] = a32 / k13["hbm_read_gbs"]
    share = {k: round(v[0] / max(prof_total_ms, 1e-9), 4) for k, v in prof.items()}
    kern = {k: {"ms": round(v[0], 3), "launches": v[1],
                "achieved": (round(v[2] / (v[0] / 1e3) / (1e12 if k.startswith("fw") else 1e9), 2) if v[0] > 0 else None),
                "unit": "Trelax/s" if k.startswith("fw") else "GB/s"} for k, v in prof.items()}

    # ---------------- per-type breakdown
    by = {}
    for kind, ms, na, info in per_update:
        by.setdefault(kind, []).append((ms, info))
    breakdown = {}
    for kind, lst in by.items():
        mss = [m for m, _ in lst]
        breakdown[kind] = {
            "count": len(lst), "ms_median": statistics.median(mss), "ms_mean": statistics.mean(mss),
            "ms_max": max(mss), "early_exit": sum(i["early_exit"] for _, i in lst),
            "paths": {str(p): sum(1 for _, i in lst if i["path"] == p) for p in sorted({i["path"] for _, i in lst})},
            "affected_pairs_median": statistics.median([i["affected_pairs"] for _, i in lst]),
        }
    all_ms = [m for _, m, _, _ in per_update]

    # ---------------- CPU baseline (oracle on the host cores, rank 0, N=1)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        Wc = synth.graph(spec)
        tp, p, n = oracle_pivot_time(Wc, budget_s=12.0)
        del Wc
        per_update_s = n * tp
        cpu = {"value": n * n / per_update_s, "unit": UNIT, "cores": cores(), "kind": "oracle",
               "sample": f"{p} Floyd-Warshall pivots of the n={n} int64 oracle matrix "
                         f"({tp * 1e3:.1f} ms/pivot), extrapolated x n: the oracle's cold recompute per update"}

    # ---------------- post-run check of the final state (test infrastructure,
    # outside every timed region): sampled rows / columns of the GPU's D after
    # all the updates vs oracle Dijkstra on the host graph
    verify = None if args.no_verify else final_check(h, hg_final, seq, rank, world, pg, dev,
                                                      args.verify_samples)
    n_final = h.n
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "int32",
            "data": "synthetic (seeded BJ.c4 graph: directed complete, U[1,1000]; seeded update sequence)",
            "config": {"workload": "BJ.c4", "n": n0, "n_final": n_final, "updates_per_step": UPDATES_PER_STEP,
                       "directed": True, "parallelism": f"row-shard x{world}" if world > 1 else "1 GPU",
                       "l2": "inputs larger than L2 (D = 4 GiB, WT = 4 GiB)",
                       "ms_per_update_median": statistics.median(all_ms),
                       "ms_per_update_mean": statistics.mean(all_ms),
                       "cold_fw_ms": cold_ms, "warm_vs_cold_speedup": cold_ms / statistics.mean(all_ms)},
            "roofline": roof,
            "roofline_int32": roof32,
            "k13": k13,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clocks,
            "kernels": kern,
            "kernel_share": share,
            "per_type": breakdown,
            "setup_s": setup_s,
            "verify": verify,
        }
        print(json.dumps(line), flush=True)
        if args.json_extra:
            with open(args.json_extra, "w") as f:
                json.dump(line, f, indent=1)
    h.close()
    if verify is not None and not verify["ok"]:
        sys.exit(3)   # the reported number was taken on a wrong state
    if pg is not None:
        pg.destroy_process_group()


if __name__ == "__main__":
    main()
