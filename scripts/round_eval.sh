# Round evaluation on one B200 (run under gpurun from the repo root).
set -x
nvidia-smi --query-gpu=name,driver_version,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 400 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 900 python scripts/bench_configs.py c1 c2 c3 c5 c4f1 > gpurun_out/configs.jsonl 2> gpurun_out/configs.err; echo "cfg rc=$?" >> gpurun_out/configs.err
timeout 300 python scripts/ncu_probe.py 32768 > gpurun_out/ncu_probe_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_detect_p8|k_detect_p16|k_sparse_phase_a|k_sparse_short|k_sparse_round|k_addcol_gather|k_addrow|k_addnode_pass1_p8|k_addnode_pass1_p16|k_rank1|k_mirror_pairs|k_query_scan|k_query_solve" -c 20 -o gpurun_out/hot_full python scripts/ncu_probe.py 32768 > gpurun_out/ncu_hot.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fw_tile3 -s 101 -c 1 -o gpurun_out/fw_full python scripts/ncu_probe.py 32768 > gpurun_out/ncu_fw.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches.csv python bench.py --no-cpu-baseline --steps 2 --warmup 3 > gpurun_out/ncu_launch.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_launch.log
python scripts/make_traffic.py gpurun_out/hot_full.ncu-rep gpurun_out/fw_full.ncu-rep > gpurun_out/traffic.json 2> gpurun_out/traffic.err
