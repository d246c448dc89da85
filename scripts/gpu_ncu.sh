#!/bin/bash
# One full ncu capture of a chosen kernel (KREGEX) on a chosen config (NCFG), short bench.
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
T=${RUN_TAG:-ncu}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-attn_fused} -s 2 -c 1 \
  -o gpurun_out/${T} python bench.py --config ${NCFG:-4} --steps 1 --warmup 3 --layers 2 --no-cpu-baseline > gpurun_out/${T}.log 2>&1
