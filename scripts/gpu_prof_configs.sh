#!/bin/bash
# ncu --set full of the pair kernel for further configs / variants (one launch each, relaxed-fluid inputs)
run() {  # tag, prof_step args...
  local tag=$1; shift
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pairs -s 1 -c 1 -o gpurun_out/prof_$tag \
    python scripts/prof_step.py "$@" > gpurun_out/ncu_$tag.log 2>&1; echo $tag=$?
}
python scripts/prof_step.py --config 4 --input fluid --cache gpurun_out/fluid_c4.npy --variant ds > /dev/null 2>&1
run c4_ds --config 4 --variant ds --input fluid --cache gpurun_out/fluid_c4.npy
rm -f gpurun_out/fluid_c4.npy
python scripts/prof_step.py --config 2 --input fluid --cache gpurun_out/fluid_c2.npy > /dev/null 2>&1
run c2_do --config 2 --variant do --input fluid --cache gpurun_out/fluid_c2.npy
python scripts/prof_step.py --config 1 --input fluid --cache gpurun_out/fluid_c1.npy > /dev/null 2>&1
run c1_do --config 1 --variant do --input fluid --cache gpurun_out/fluid_c1.npy
run c1_do_f64 --config 1 --variant do --prec f64 --input fluid --cache gpurun_out/fluid_c1.npy
run c0_do_f64 --config 0 --variant do --prec f64
