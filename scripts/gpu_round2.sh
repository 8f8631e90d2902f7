#!/bin/bash
# Round-2 evidence cycle: GPU tests, smoke, default bench line (C4 DO fluid + cpu baseline), per-config lines,
# the reference arm, ncu launch list of the bench, ncu --set full of k_pairs (C4 DO) and the sparse-cell
# kernel (C3 DO), both on the bench's relaxed-fluid input.
TAG=${1:-r02}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo pytest_exit=$?; tail -2 gpurun_out/pytest_gpu_$TAG.log
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/smoke_$TAG.log 2>&1; echo smoke_exit=$?
timeout 900 python bench.py > gpurun_out/bench_$TAG.log 2>&1; echo bench_exit=$?; tail -1 gpurun_out/bench_$TAG.log | cut -c1-400
for c in 0 1 2 3 4; do for v in do ds; do
  timeout 600 python bench.py --config $c --variant $v --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_${TAG}_c${c}_${v}.log 2>&1; echo c${c}_${v}=$?
done; done
timeout 600 python bench.py --config 4 --variant do --input lattice --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_${TAG}_c4_do_lattice.log 2>&1; echo lattice=$?
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_${TAG}_ref.log 2>&1; echo ref_exit=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_launch_$TAG.log 2>&1; echo ncul_exit=$?
for c in 4 3; do
  python scripts/prof_step.py --config $c --input fluid --cache gpurun_out/fluid_c$c.npy > /dev/null 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pairs -s 1 -c 1 -o gpurun_out/prof_${TAG}_c$c \
    python scripts/prof_step.py --config $c --input fluid --cache gpurun_out/fluid_c$c.npy > gpurun_out/ncu_${TAG}_c$c.log 2>&1; echo ncu_c${c}_exit=$?
  rm -f gpurun_out/fluid_c$c.npy
done
