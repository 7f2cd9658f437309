#!/bin/bash
# Like sweep.sh, for the 4-byte streams: per variant, bench.py's int32 leg
# (mirror off, SURVEY §8(d-4) bytes) — the per-class event times and GB/s of
# `roofline_int32`.
for spec in "$@"; do
  label="${spec%%=*}"; flags="${spec#*=}"
  APSP_NVCC_EXTRA="$flags" python paper_2412_15122_b200/build.py --force > /dev/null 2> gpurun_out/sweepi_build_$label.err || { echo "$label BUILD FAILED"; continue; }
  timeout 400 python bench.py --steps 2 --warmup 2 --no-e2e --no-verify --no-cpu-baseline --no-cold \
      > gpurun_out/sweepi_$label.json 2> gpurun_out/sweepi_$label.err
  python - "$label" <<'PY'
import json, sys
label = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/sweepi_{label}.json").read().strip().splitlines()[-1])
except Exception as e:
    print(label, "FAILED", e); sys.exit()
ri = d["roofline_int32"]
print(label, f"{d['value']:.3e}", json.dumps({c: (v["ms"], v["launches"], v["achieved_gbs"]) for c, v in ri["classes"].items()}))
PY
done
