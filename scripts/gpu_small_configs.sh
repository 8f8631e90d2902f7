#!/bin/bash
# per-config bench lines of the small configs (C0-C2, both variants) into gpurun_out/bench_${TAG}_c*.log
TAG=${1:-small}
for c in 0 1 2; do for v in do ds; do
  timeout 600 python bench.py --config $c --variant $v --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_${TAG}_c${c}_${v}.log 2>&1; echo c${c}_${v}=$?
done; done
