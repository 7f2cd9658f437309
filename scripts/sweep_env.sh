#!/bin/bash
# Runtime-knob sweep on one B200 (run under gpurun from the repo root):
#   scripts/sweep_env.sh "<label>=<VAR=value ...>" ...
# For each variant: a short bench.py with those environment variables set,
# printing the per-class kernel times and per-type update medians.
for spec in "$@"; do
  label="${spec%%=*}"; vars="${spec#*=}"
  env $vars timeout 300 python bench.py --steps 2 --warmup 2 --no-e2e --no-int32 --no-verify --no-cpu-baseline \
      > gpurun_out/sweepe_$label.json 2> gpurun_out/sweepe_$label.err
  python - "$label" <<'PY'
import json, sys
label = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/sweepe_{label}.json").read().strip().splitlines()[-1])
except Exception as e:
    print(label, "FAILED", e); sys.exit()
k = {c: (round(v["ms"], 2), v["launches"]) for c, v in d["kernels"].items() if v["launches"]}
pt = {t: round(v["ms_median"], 4) for t, v in d["per_type"].items()}
print(label, f"{d['value']:.3e}", round(d["ms_per_step"], 3), pt, json.dumps(k))
PY
done
