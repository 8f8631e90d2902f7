#!/bin/bash
# ncu --set full of k_pairs on C4 DO (relaxed fluid), one launch
python scripts/prof_step.py --config 4 --input fluid --cache gpurun_out/fluid_c4.npy > /dev/null 2>&1
TAG=${TAG:-c4}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pairs -s 1 -c 1 -o gpurun_out/prof_$TAG \
  python scripts/prof_step.py --config 4 --input fluid --cache gpurun_out/fluid_c4.npy > gpurun_out/ncu_$TAG.log 2>&1; echo ncu=$?
rm -f gpurun_out/fluid_c4.npy
