#!/bin/bash
timeout 900 env NC_K3=2 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_v4.log 2>&1; echo pytest_v4=$?; tail -2 gpurun_out/pytest_v4.log
for lib in "$@"; do
  NC_K3=2 NC_LIB=exp/lib_$lib.so timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu > gpurun_out/sweep_$lib.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/sweep_$lib.log').read().strip().splitlines()[-1]); r=d['roofline']
print('$lib pairs_ms %.2f ms/step %.2f' % (r['kernel_ms'], d['ms_per_step']))" 2>/dev/null || { echo "$lib failed"; tail -3 gpurun_out/sweep_$lib.log; }
done
