#!/bin/bash
# smoke(), the reference arm, and one bench line per BASELINE config x variant (config precision)
TAG=${1:-cfg}
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke_$TAG.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref_$TAG.log 2>&1; echo ref=$?; tail -1 gpurun_out/ref_$TAG.log | cut -c1-300
for c in 0 1 2 3 4; do for v in do ds; do
  timeout 600 python bench.py --config $c --variant $v --steps 10 --warmup 3 $( [ $c = 4 ] && [ $v = do ] || echo --no-cpu ) > gpurun_out/bench_${TAG}_c${c}_${v}.log 2>&1
  python - gpurun_out/bench_${TAG}_c${c}_${v}.log <<'PY'
import json,sys
f=sys.argv[1]
try:
    d=json.loads(open(f).read().strip().splitlines()[-1]); r=d['roofline']
    print("%s %s %s ms/step %.3f pairs_ms %.3f value %.3g psteps %.3g frac %.3f kern %s" % (d['config']['workload'], d['config']['variant'], d['dtype'], d['ms_per_step'], r['kernel_ms'], d['value'], d['particle_steps_per_s'], r['frac'], r.get('pair_kernel')))
except Exception as e:
    print(f, "FAIL", open(f).read()[-400:])
PY
done; done
