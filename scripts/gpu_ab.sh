#!/bin/bash
# A/B cycle: GPU parity tests with the default kernel, then bench of both fp32 pair kernels (NC_K3=1 old, 2 new)
TAG=${1:-ab}
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_$TAG.log 2>&1; echo pytest_exit=$?; tail -15 gpurun_out/pytest_$TAG.log
for v in 2 1; do
NC_K3=$v timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_${TAG}_k$v.log 2>&1; echo bench_k$v=$?
python -c "
import json; d=json.loads(open('gpurun_out/bench_${TAG}_k$v.log').read().strip().splitlines()[-1]); r=d['roofline']
print('K3=$v value %.4g ms/step %.2f pairs_ms %.2f frac %.3f' % (d['value'], d['ms_per_step'], r['kernel_ms'], r['frac']))" || tail -5 gpurun_out/bench_${TAG}_k$v.log
done
