#!/bin/bash
# ncu --set full of the sparse-cell pair kernels on C3 DO (relaxed fluid)
python scripts/prof_step.py --config 3 --input fluid --cache gpurun_out/fluid_c3.npy > /dev/null 2>&1
for k in ${KERNELS:-rows sparse}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pairs -s 1 -c 1 -o gpurun_out/prof_${k}_c3 \
    python scripts/prof_step.py --config 3 --input fluid --cache gpurun_out/fluid_c3.npy --pair-kernel $k > gpurun_out/ncu_${k}_c3.log 2>&1; echo ncu_${k}=$?
done
rm -f gpurun_out/fluid_c3.npy
