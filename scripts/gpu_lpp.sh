#!/bin/bash
# small-system kernels: sparse kernel with 1 / 4 threads per particle vs segment / rows; then the sparse tests with LPP=4
for l in 1 4; do NC_SP_LPP=$l timeout 300 python scripts/small_kernel_probe.py; done
NC_SP_LPP=4 timeout 900 python -m pytest tests -m gpu -q -x -k "sparse or c1_both or cutoff or truncated or edge or slab" > gpurun_out/pytest_lpp4.log 2>&1; echo pytest_lpp4=$?; tail -3 gpurun_out/pytest_lpp4.log
