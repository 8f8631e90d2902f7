#!/bin/bash
for s in C1 E2; do
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_small_$s.csv python scripts/small_steps.py $s > /dev/null 2>&1; echo $s=$?
python scripts/launch_share.py gpurun_out/launches_small_$s.csv
done
