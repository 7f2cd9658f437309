"""Summarise ncu reports into small JSON files for profiles/ (read here, no GPU).

    python scripts/ncu_summary.py OUT.json REPORT.ncu-rep [REPORT2.ncu-rep ...]

Per captured launch: duration, DRAM bytes read/written, DRAM and L2
throughput, SM / ALU-pipe utilisation, occupancy, registers, grid, and the
top warp-stall reasons.
"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_peak",
    "lts__t_bytes.sum": "l2_bytes",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "alu_pipe_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "smsp__inst_executed.sum": "inst_executed",
    "sm__cycles_elapsed.avg.per_second": "sm_clock",
}


def raw(report):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main():
    dst, reports = sys.argv[1], sys.argv[2:]
    res = []
    for rep in reports:
        hdr, units, rows = raw(rep)
        for r in rows:
            d = {"report": rep.split("/")[-1], "kernel": r[hdr.index("Kernel Name")].split("(")[0]}
            for k, name in KEYS.items():
                if k in hdr:
                    d[name] = f"{r[hdr.index(k)]} {units[hdr.index(k)]}".strip()
            stalls = []
            for i, h in enumerate(hdr):
                pre, suf = "smsp__average_warps_issue_stalled_", "_per_issue_active.ratio"
                if h.startswith(pre) and h.endswith(suf):
                    try:
                        stalls.append((float(r[i].replace(",", "")), h[len(pre):-len(suf)]))
                    except ValueError:
                        pass
            d["top_stalls"] = [[round(v, 2), k] for v, k in sorted(stalls, reverse=True)[:5]]
            res.append(d)
    with open(dst, "w") as f:
        json.dump(res, f, indent=1)
    for d in res:
        print(d["kernel"], d.get("duration"), d.get("dram_read"), d.get("dram_pct_peak"))


if __name__ == "__main__":
    main()
