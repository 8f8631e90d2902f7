# ncu --set full of one C4 DO k_pairs launch on the relaxed-fluid input (the bench's input)
TAG=${1:-c4f}
python scripts/prof_step.py --input fluid --cache gpurun_out/fluid_c4_do.npy > gpurun_out/prof_${TAG}_prep.log 2>&1; echo prep=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pairs -s 1 -c 1 -o gpurun_out/prof_${TAG} \
  python scripts/prof_step.py --input fluid --cache gpurun_out/fluid_c4_do.npy > gpurun_out/ncu_${TAG}.log 2>&1; echo ncu=$?
rm -f gpurun_out/fluid_c4_do.npy
