#!/bin/bash
# Compile-time variant sweep on one B200 (run under gpurun from the repo root):
#   scripts/sweep.sh "<label>=<nvcc -D flags>" ...
# For each variant: rebuild libapsp_warm.so with the flags, run a short
# bench.py and print the per-class kernel times (the library's own CUDA-event
# profile) and the per-type update medians.
for spec in "$@"; do
  label="${spec%%=*}"; flags="${spec#*=}"
  APSP_NVCC_EXTRA="$flags" python paper_2412_15122_b200/build.py --force > /dev/null 2> gpurun_out/sweep_build_$label.err || { echo "$label BUILD FAILED"; continue; }
  timeout 300 python bench.py --steps 2 --warmup 2 --no-e2e --no-int32 --no-verify --no-cpu-baseline --no-cold \
      > gpurun_out/sweep_$label.json 2> gpurun_out/sweep_$label.err
  python - "$label" <<'PY'
import json, sys
label = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/sweep_{label}.json").read().strip().splitlines()[-1])
except Exception as e:
    print(label, "FAILED", e); sys.exit()
k = {c: (v["ms"], v["launches"], v["achieved"]) for c, v in d["kernels"].items() if v["launches"]}
pt = {t: round(v["ms_median"], 4) for t, v in d["per_type"].items()}
print(label, f"{d['value']:.3e}", round(d["ms_per_step"], 3), pt, json.dumps(k))
PY
done
