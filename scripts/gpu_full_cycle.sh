set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_full.log 2>&1; echo pytest_exit=$?; tail -3 gpurun_out/pytest_gpu_full.log
timeout 600 python bench.py > gpurun_out/bench_default.log 2>&1; echo bench_exit=$?; tail -1 gpurun_out/bench_default.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/ncu_launch.log 2>&1; echo ncul_exit=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pairs -s 1 -c 1 -o gpurun_out/prof_cur python scripts/prof_step.py > gpurun_out/ncu_cur.log 2>&1; echo ncu_exit=$?
