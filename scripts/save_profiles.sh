#!/bin/bash
# Copy one round_eval.sh run (gpurun_out/) into profiles/ under the round's
# prefix (run here, after the gpurun call merged its outputs):
#   scripts/save_profiles.sh r02
set -e
R=${1:?round prefix, e.g. r02}
G=gpurun_out
P=profiles
tail -1 $G/bench.log > /dev/null
grep '^{' $G/bench.log | tail -1 > $P/${R}_bench.json
cp $G/configs.jsonl $P/${R}_configs.jsonl
cp $G/launches.csv $P/${R}_launches_timed.csv
python scripts/launch_summary.py $G/launches.csv $P/${R}_launch_summary.json \
  "python bench.py --steps 2 --warmup 3 --no-e2e --no-int32 --no-verify --no-cpu-baseline (NVTX range timed)" > /dev/null
cp $G/ncu_hot_kernels.json $P/${R}_ncu_hot_kernels.json
cp $G/ncu_int32_streams.json $P/${R}_ncu_int32_streams.json
cp $G/ncu_fp32_streams.json $P/${R}_ncu_fp32_streams.json
cp $G/traffic.json $P/traffic.json
cp $G/smi.txt $P/${R}_smi.txt
scripts/sass_tma.sh > $P/${R}_sass_tma.txt
ls -la $P | grep "$R"
