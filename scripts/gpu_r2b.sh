#!/bin/bash
# Microbenchmarks (MUFU / TMA), per-tile pipeline trace (PB_TILE_TRACE variant), page-mover
# bench, ncu launch list + full captures of the fused kernel (cfg4), the page movers and the
# swap kernels (cfg5).
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
T=${RUN_TAG:-r2b}
timeout 300 ./scripts/microbench/tma_mufu > gpurun_out/${T}_micro.txt 2>&1
SO=paper_2312_05516_b200/libpensieve_b200.so
cp $SO /tmp/pb_base.so
cp paper_2312_05516_b200/variants/tt.so $SO
timeout 300 python scripts/trace_tiles.py 4 > gpurun_out/${T}_trace_tiles.txt 2>&1
cp /tmp/pb_base.so $SO
timeout 300 python scripts/bench_page_copy.py > gpurun_out/${T}_page_copy.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:attn -c 40 --csv \
  --log-file gpurun_out/${T}_launches_cfg4.csv python bench.py --steps 1 --warmup 3 --layers 4 --no-cpu-baseline --no-subconfigs > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fused -s 2 -c 1 \
  -o gpurun_out/${T}_fused python bench.py --steps 1 --warmup 3 --layers 2 --no-cpu-baseline --no-subconfigs > gpurun_out/${T}_ncu_fused.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:page_copy -c 2 \
  -o gpurun_out/${T}_page_copy python scripts/bench_page_copy.py 4096 1024 1 > gpurun_out/${T}_ncu_pc.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:swap_ -s 6 -c 4 \
  -o gpurun_out/${T}_swap python bench.py --config 5 --steps 2 --warmup 3 > gpurun_out/${T}_ncu_swap.log 2>&1
