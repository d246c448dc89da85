#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_swap_gpu.py -q -x 2>&1 | tail -20 > gpurun_out/r12_swap.txt
CASES="d1 d2 d3 d4 mix cfg3 cfg2" CFGS="3 2 4" NO_PYTEST=1 RUN_TAG=r12 bash scripts/gpu_quick.sh
