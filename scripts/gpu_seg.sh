#!/bin/bash
# sparse-cell kernel: GPU parity tests, then C1/C3 bench lines with NC_SEG=1 (segment kernel) vs NC_SEG=0
TAG=${1:-seg}
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_$TAG.log 2>&1; echo pytest_exit=$?; tail -4 gpurun_out/pytest_$TAG.log
for cfg in 3 1; do for v in do ds; do for sg in 1 0; do
NC_SEG=$sg timeout 300 python bench.py --config $cfg --variant $v --steps 20 --warmup 3 --no-cpu > gpurun_out/bench_${TAG}_c${cfg}_${v}_s$sg.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/bench_${TAG}_c${cfg}_${v}_s$sg.log').read().strip().splitlines()[-1]); r=d['roofline']
print('C$cfg $v seg=$sg ms/step %.3f pairs_ms %.3f value %.3g' % (d['ms_per_step'], r['kernel_ms'], d['value']), {k: round(x,3) for k,x in d['kernel_ms_per_step'].items()})" 2>/dev/null || { echo "C$cfg $v seg=$sg failed"; tail -3 gpurun_out/bench_${TAG}_c${cfg}_${v}_s$sg.log; }
done; done; done
