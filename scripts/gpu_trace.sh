#!/bin/bash
# per-tile pipeline traces (trace builds: scripts/build_variants.sh tt "-DPB_TILE_TRACE=1" ...)
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
T=${RUN_TAG:-trace}
SO=paper_2312_05516_b200/libpensieve_b200.so
cp $SO /tmp/pb_base.so
for v in ${VARIANTS:-tt}; do
  cp paper_2312_05516_b200/variants/$v.so $SO
  echo "== $v $(timeout 300 python scripts/trace_tiles.py ${CFG:-4} 2>&1 | tail -1)" >> gpurun_out/${T}_trace.txt
done
cp /tmp/pb_base.so $SO
