"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel.

    python scripts/launch_summary.py launches.csv OUT.json "command that was profiled"
"""
import csv
import json
import sys
from collections import defaultdict


def main():
    src, dst, cmd = sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else ""
    rows = [r for r in csv.reader(open(src)) if len(r) > 5]
    hdr, data = rows[0], rows[1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    ms = defaultdict(float)
    cnt = defaultdict(int)
    for r in data:
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}.get(r[ui], 1e-6)
        k = r[ki].split("(")[0].replace("void ", "").replace("apsp::", "")
        ms[k] += float(r[vi].replace(",", "")) * scale
        cnt[k] += 1
    total = sum(ms.values())
    out = {"command": cmd, "total_ms": round(total, 3), "launches": sum(cnt.values()),
           "by_kernel": [{"kernel": k, "launches": cnt[k], "ms": round(v, 3), "pct": round(100 * v / total, 2)}
                         for k, v in sorted(ms.items(), key=lambda kv: -kv[1])]}
    with open(dst, "w") as f:
        json.dump(out, f, indent=1)
    for e in out["by_kernel"][:12]:
        print(f"{e['pct']:6.2f}% {e['ms']:10.3f} ms {e['launches']:6d}  {e['kernel']}")


if __name__ == "__main__":
    main()
