#!/bin/bash
# Evidence pass: default bench line (config 4, with the CPU reference baseline), the other
# configs, an ncu launch list of the default bench, and one full ncu capture per hot kernel.
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
T=${RUN_TAG:-prof}
nproc > gpurun_out/${T}_nproc.txt
timeout 900 python bench.py > gpurun_out/${T}_bench_default.txt 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${T}_bench_reference.txt 2>&1
for c in 2 3; do timeout 600 python bench.py --config $c > gpurun_out/${T}_bench_cfg$c.txt 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:attn -c 40 --csv \
  --log-file gpurun_out/${T}_launches_cfg4.csv python bench.py --steps 1 --warmup 3 --layers 8 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:attn -c 40 --csv \
  --log-file gpurun_out/${T}_launches_cfg3.csv python bench.py --config 3 --steps 1 --warmup 3 --layers 8 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fused -s 2 -c 1 \
  -o gpurun_out/${T}_prefill python bench.py --steps 1 --warmup 3 --layers 2 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_decode -s 2 -c 1 \
  -o gpurun_out/${T}_decode python bench.py --config 3 --steps 1 --warmup 3 --layers 2 --no-cpu-baseline > /dev/null 2>&1
