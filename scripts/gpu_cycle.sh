#!/bin/bash
# one GPU iteration: parity tests (not C4), bench, ncu of k_pairs on C4.  Usage: scripts/gpu_cycle.sh TAG [noprof]
TAG=${1:-x}
timeout 900 python -m pytest tests -m gpu -q -x -k "not c4" > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo pytest_exit=$?; tail -3 gpurun_out/pytest_gpu_$TAG.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_$TAG.log 2>&1; echo bench_exit=$?
python -c "
import json; d=json.loads(open('gpurun_out/bench_$TAG.log').read().strip().splitlines()[-1]); r=d['roofline']
print('value %.4g ms/step %.2f pairs_ms %.2f frac %.3f e2e %.4g' % (d['value'], d['ms_per_step'], r['kernel_ms'], r['frac'], d['e2e']['value'])); print(d['kernel_ms_per_step'])"
if [ "$2" != "noprof" ]; then
python scripts/prof_step.py > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_pairs -s 1 -c 1 -o gpurun_out/prof_$TAG python scripts/prof_step.py > gpurun_out/ncu_$TAG.log 2>&1; echo ncu_exit=$?
fi
