#!/bin/bash
# ncu --set full of one k_pairs* launch on C4 DO (after a plain run exits 0). Usage: scripts/gpu_prof.sh TAG [extra prof_step args]
TAG=${1:-x}; shift
timeout 300 python scripts/prof_step.py "$@" > gpurun_out/plain_$TAG.log 2>&1 || { echo plain_failed; tail gpurun_out/plain_$TAG.log; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pairs -s 1 -c 1 -o gpurun_out/prof_$TAG python scripts/prof_step.py "$@" > gpurun_out/ncu_$TAG.log 2>&1; echo ncu_exit=$?
