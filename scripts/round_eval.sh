#!/bin/bash
# Round evaluation on one B200 (run under gpurun from the repo root): the bench
# line, per-config measurements, the timed region's launch list and full ncu
# captures of the hot kernels — the int8-mirror path bench.py times, the
# int32 (4 B/entry) streams and the fp32 streams (each ncu command after its
# plain run exited 0).
set -x
nvidia-smi --query-gpu=name,driver_version,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 900 python scripts/bench_configs.py c1 c2 c3 c5 c4f1 > gpurun_out/configs.jsonl 2> gpurun_out/configs.err; echo "cfg rc=$?" >> gpurun_out/configs.err
# launch list of bench.py's timed region only (NVTX range "timed")
timeout 300 python bench.py --steps 2 --warmup 3 --no-e2e --no-int32 --no-verify --no-cpu-baseline > gpurun_out/bench_short.log 2>&1 && \
  timeout 900 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-int32 --no-verify --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 300 python scripts/ncu_probe.py 32768 > gpurun_out/ncu_probe_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_detect_p8|k_phase_a0|k_sparse_phase_aq|k_sparse_short|k_sparse_full|k_sparse_rounds_coop|k_addcol_mt|k_addrow|k_rank1_p8|k_validate_vec|k_query_scan|k_query_solve|k_update_prep" -c 20 -o gpurun_out/hot_full python scripts/ncu_probe.py 32768 > gpurun_out/ncu_hot.log 2>&1
python scripts/make_traffic.py gpurun_out/hot_full.ncu-rep > gpurun_out/traffic.json 2> gpurun_out/traffic.err
python scripts/ncu_summary.py gpurun_out/ncu_hot_kernels.json gpurun_out/hot_full.ncu-rep > gpurun_out/ncu_sum.log 2>&1
# the 4-byte streams (mirror off) and fp32, n = 32768: detection, pass 1, rank-1
timeout 300 python scripts/ncu_probe.py 32768 --no-mirror > gpurun_out/ncu_probe_i32_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none -k regex:"k_detect_stream|k_addnode_pass1|k_rank1" -c 12 -o gpurun_out/i32_full python scripts/ncu_probe.py 32768 --no-mirror > gpurun_out/ncu_i32.log 2>&1
timeout 300 python scripts/ncu_probe.py 32768 --fp32 > gpurun_out/ncu_probe_f32_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none -k regex:"k_detect_stream|k_addnode_pass1|k_rank1" -c 12 -o gpurun_out/f32_full python scripts/ncu_probe.py 32768 --fp32 > gpurun_out/ncu_f32.log 2>&1
python scripts/ncu_summary.py gpurun_out/ncu_int32_streams.json gpurun_out/i32_full.ncu-rep >> gpurun_out/ncu_sum.log 2>&1
python scripts/ncu_summary.py gpurun_out/ncu_fp32_streams.json gpurun_out/f32_full.ncu-rep >> gpurun_out/ncu_sum.log 2>&1
# gpurun copies back at most 64 MiB: keep the hot-kernel report, summaries of the others
rm -f gpurun_out/i32_full.ncu-rep gpurun_out/f32_full.ncu-rep
ls -la gpurun_out > gpurun_out/ls.txt
