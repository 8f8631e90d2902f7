#!/bin/bash
# rows-kernel cycle: its GPU tests, then C3 / C1 lines with each sparse-cell kernel (pair kernel ms)
timeout 900 python -m pytest tests -m gpu -q -x -k "rows or sparse or segment or cutoff or truncated" > gpurun_out/pytest_rows.log 2>&1; echo pytest_exit=$?; tail -15 gpurun_out/pytest_rows.log
for v in do ds; do for k in ${KS:-sparse rows}; do
timeout 300 python bench.py --pair-kernel $k --config 3 --variant $v --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_rows_c3_${v}_$k.log 2>&1; echo c3_${v}_$k=$?
python -c "
import json; d=json.loads(open('gpurun_out/bench_rows_c3_${v}_$k.log').read().strip().splitlines()[-1]); r=d['roofline']
print('$v $k ms/step %.4f pairs_ms %.4f kernel %s' % (d['ms_per_step'], r['kernel_ms'], r.get('pair_kernel')))" || tail -3 gpurun_out/bench_rows_c3_${v}_$k.log
done; done
