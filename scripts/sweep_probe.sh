#!/bin/bash
# Compile-time variant sweep of one tight increase (scripts/update_probe.py)
# on one B200 (run under gpurun from the repo root):
#   scripts/sweep_probe.sh <c2|c5> "<label>=<nvcc -D flags>[;ENV=VAL ...]" ...
# Per variant: rebuild, then the probe's launch list (ncu, gpu__time_duration
# only) and its event-timed total.
cfg=$1; shift
for spec in "$@"; do
  label="${spec%%=*}"; rest="${spec#*=}"; flags="${rest%%;*}"; envs=""
  [[ "$rest" == *";"* ]] && envs="${rest#*;}"
  APSP_NVCC_EXTRA="$flags" python paper_2412_15122_b200/build.py --force > /dev/null 2> gpurun_out/sp_build_$label.err || { echo "$label BUILD FAILED"; continue; }
  env $envs timeout 300 python scripts/update_probe.py $cfg > gpurun_out/sp_$label.log 2>&1
  env $envs timeout 600 ncu --nvtx --nvtx-include "probe/" --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/sp_$label.csv python scripts/update_probe.py $cfg > /dev/null 2>&1
  python - "$label" <<'PY'
import csv, sys
label = sys.argv[1]
tot = open(f"gpurun_out/sp_{label}.log").read().split("\n")
try:
    rows = [r for r in csv.reader(open(f"gpurun_out/sp_{label}.csv")) if len(r) > 5]
    h = rows[0]
    ks = [(r[h.index("Kernel Name")].split("<")[0].split("(")[0].replace("void ", ""), float(r[h.index("Metric Value")].replace(",", "")) / 1e3) for r in rows[1:]]
except Exception as e:
    ks = [("?", 0.0)]
print(label, [l.split("{")[0] for l in tot if l][-2:], " ".join(f"{k}:{v:.1f}" for k, v in ks if v > 3))
PY
done
