#!/bin/bash
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_v0.log 2>&1; echo pytest_exit=$?; tail -2 gpurun_out/pytest_gpu_v0.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_v0.log 2>&1; echo smoke_exit=$?
timeout 900 python bench.py --no-cpu > gpurun_out/bench_v0.log 2>&1; echo bench_exit=$?; tail -1 gpurun_out/bench_v0.log | cut -c1-300
