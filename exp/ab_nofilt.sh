#!/bin/bash
# phase timing: setup/staging-only builds (K3_SKIP=1) of the q48 baseline vs the TMA+prefetch version
for v in q48 q48nf new newnf; do
  NC_LIB=exp/lib_$v.so timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu > gpurun_out/ab_$v.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/ab_$v.log').read().strip().splitlines()[-1]); r=d['roofline']
print('$v pairs_ms %.2f' % r['kernel_ms'])" 2>/dev/null || echo "$v failed"
done
