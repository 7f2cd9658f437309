#!/bin/bash
# Like sweep.sh, plus BJ.c2's tight increase (scripts/update_probe.py c2
# --bench-edge) per variant: scripts/sweep_c2.sh "<label>=<nvcc -D flags>" ...
for spec in "$@"; do
  label="${spec%%=*}"; flags="${spec#*=}"
  APSP_NVCC_EXTRA="$flags" python paper_2412_15122_b200/build.py --force > /dev/null 2> gpurun_out/sweep_build_$label.err || { echo "$label BUILD FAILED"; continue; }
  echo "$label c2: $(timeout 300 python scripts/update_probe.py c2 --bench-edge 2>&1 | tail -1 | cut -c1-60)"
  bash scripts/sweep.sh "$label=$flags" 2>&1 | cut -c1-400
done
