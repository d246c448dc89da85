#!/bin/bash
# Round-2 evidence for the page movers / swaps and the external yardstick:
#  flashinfer trtllm-gen sm100 paged kernels vs ours on cfg2/3/4; page-mover bench; ncu full
#  captures of page_copy_kernel and the swap gather/scatter kernels (cfg5); cfg5 bench line.
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
T=${RUN_TAG:-r2z}
timeout 900 python scripts/bench_flashinfer.py --configs 2,3,4 --reps 20 --out gpurun_out/${T}_flashinfer.json > gpurun_out/${T}_flashinfer.txt 2>&1
timeout 300 python scripts/bench_page_copy.py > gpurun_out/${T}_page_copy.txt 2>&1
timeout 600 python bench.py --config 5 --no-cpu-baseline > gpurun_out/${T}_cfg5.txt 2>&1
timeout 600 ncu --set full --clock-control none -k regex:page_copy -c 2 \
  -o gpurun_out/${T}_page_copy python scripts/bench_page_copy.py 4096 1024 1 > gpurun_out/${T}_ncu_pc.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:swap_ -s 6 -c 4 \
  -o gpurun_out/${T}_swap python bench.py --config 5 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_ncu_swap.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:swap_ -c 60 --csv \
  --log-file gpurun_out/${T}_launches_swap.csv python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
