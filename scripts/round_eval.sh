set -x
nvidia-smi --query-gpu=name,driver_version,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 400 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 900 python scripts/bench_configs.py c1 c2 c3 c5 c4f1 > gpurun_out/configs.jsonl 2> gpurun_out/configs.err; echo "cfg rc=$?" >> gpurun_out/configs.err
timeout 300 python scripts/query_probe.py 32768 0 > gpurun_out/qp.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches.csv python bench.py --no-cpu-baseline --steps 2 --warmup 3 > gpurun_out/ncu_launch.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_launch.log
