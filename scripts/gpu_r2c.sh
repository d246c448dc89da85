#!/bin/bash
# r2b + fused-launch CTA timeline (cfg4) + flashinfer trtllm-gen yardstick
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
T=${RUN_TAG:-r2c}
timeout 300 python scripts/trace_fused.py 4 > gpurun_out/${T}_trace_fused4.txt 2>&1
timeout 900 python scripts/bench_flashinfer.py --out gpurun_out/${T}_flashinfer.json > gpurun_out/${T}_flashinfer.txt 2>&1
RUN_TAG=$T bash scripts/gpu_r2b.sh
