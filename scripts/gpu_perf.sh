#!/bin/bash
# Perf pass: bench lines for configs 4 (default), 2, 3; ncu launch list; one full ncu capture
# of the prefill-tile kernel and of the decode kernel.
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
T=${RUN_TAG:-perf}
timeout 900 python bench.py > gpurun_out/${T}_bench_cfg4.txt 2>&1
timeout 600 python bench.py --config 2 --no-cpu-baseline > gpurun_out/${T}_bench_cfg2.txt 2>&1
timeout 600 python bench.py --config 3 --no-cpu-baseline > gpurun_out/${T}_bench_cfg3.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:attn -c 60 --csv \
  --log-file gpurun_out/${T}_launches_cfg4.csv python bench.py --steps 1 --warmup 3 --layers 4 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_fused -s 2 -c 1 \
  -o gpurun_out/${T}_prefill python bench.py --steps 1 --warmup 3 --layers 2 --no-cpu-baseline > gpurun_out/${T}_ncu_prefill.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_decode -s 2 -c 1 \
  -o gpurun_out/${T}_decode python bench.py --config 3 --steps 1 --warmup 3 --layers 2 --no-cpu-baseline > gpurun_out/${T}_ncu_decode.log 2>&1
