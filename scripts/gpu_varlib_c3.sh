#!/bin/bash
# A/B of builds (varlib/*.so via NC_LIB) on C3 (bench lines, pair-kernel ms)
for rep in 1 2; do for v in ${VS:-do ds}; do for lib in varlib/*.so; do
NC_LIB=$lib timeout 300 python bench.py --config 3 --variant $v --steps 10 --warmup 3 --no-cpu ${EXTRA} > gpurun_out/vl.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/vl.log').read().strip().splitlines()[-1]); r=d['roofline']
print('$lib $v ms/step %.4f pairs_ms %.4f %s' % (d['ms_per_step'], r['kernel_ms'], r.get('pair_kernel')))" || tail -3 gpurun_out/vl.log
done; done; done
