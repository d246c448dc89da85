#!/bin/bash
# Tile-pipeline diagnostics: MUFU/MMA/TMA microbenchmarks, tile-bounds per variant (exp2 on
# the FMA pipe for 1 pair in N; ablations), per-tile trace, 16-layer bench per variant.
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
T=${RUN_TAG:-r2j}
SO=paper_2312_05516_b200/libpensieve_b200.so
cp $SO /tmp/pb_base.so
for b in tma_mufu mma_rate xu_mix; do
  echo "== $b" >> gpurun_out/${T}_micro.txt
  (cd scripts/microbench && timeout 120 ./$b) >> gpurun_out/${T}_micro.txt 2>&1
done
for v in ${VARIANTS:-base p4 p3 p2 a1 a2}; do
  if [ "$v" = "base" ]; then cp /tmp/pb_base.so $SO; else cp paper_2312_05516_b200/variants/$v.so $SO; fi
  echo "== $v $(timeout 300 python scripts/exp_tile_bounds.py 10 2>&1 | tail -1)" >> gpurun_out/${T}_bounds.txt
done
if [ -f paper_2312_05516_b200/variants/tt.so ]; then
  cp paper_2312_05516_b200/variants/tt.so $SO
  timeout 300 python scripts/trace_tiles.py 4 > gpurun_out/${T}_trace.txt 2>&1
fi
for v in ${BENCHV:-base p4 p3}; do
  if [ "$v" = "base" ]; then cp /tmp/pb_base.so $SO; else cp paper_2312_05516_b200/variants/$v.so $SO; fi
  echo "== $v $(timeout 300 python bench.py --steps 5 --warmup 3 --layers 16 --no-cpu-baseline --no-subconfigs 2>&1 | tail -1)" >> gpurun_out/${T}_bench.txt
done
cp /tmp/pb_base.so $SO
