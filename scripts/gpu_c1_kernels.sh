#!/bin/bash
# C1 (32k WCA) with each fp32 pair kernel: step and pair-kernel time
for v in do ds; do for k in segment sparse rows cell; do
timeout 300 python bench.py --config 1 --variant $v --steps 20 --warmup 5 --no-cpu --pair-kernel $k > gpurun_out/c1k.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/c1k.log').read().strip().splitlines()[-1]); r=d['roofline']
print('C1 $v $k ms/step %.4f pairs_ms %.4f %s launches %s' % (d['ms_per_step'], r['kernel_ms'], r.get('pair_kernel'), d.get('gpu_launches')))" || tail -3 gpurun_out/c1k.log
done; done
