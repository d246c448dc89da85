#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
for a in 0 1 2; do
  PB_ABLATE=$a timeout 300 python bench.py --steps 5 --warmup 3 --layers 16 --no-cpu-baseline > gpurun_out/r17_ablate$a.txt 2>&1
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:attn -c 20 --csv --log-file gpurun_out/r17_launches.csv python bench.py --steps 1 --warmup 3 --layers 4 --no-cpu-baseline > /dev/null 2>&1
