#!/bin/bash
# variant sweep on the tile bounds experiment (+ the per-tile trace build)
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
T=${RUN_TAG:-r2f}
SO=paper_2312_05516_b200/libpensieve_b200.so
cp $SO /tmp/pb_base.so
for v in ${VARIANTS:-base a1 a2 p4 p3 p2}; do
  if [ "$v" = "base" ]; then cp /tmp/pb_base.so $SO; else cp paper_2312_05516_b200/variants/$v.so $SO; fi
  echo "== $v" >> gpurun_out/${T}_bounds.txt
  timeout 300 python scripts/exp_tile_bounds.py 10 >> gpurun_out/${T}_bounds.txt 2>&1
done
cp paper_2312_05516_b200/variants/tt.so $SO
timeout 300 python scripts/trace_tiles.py 4 > gpurun_out/${T}_trace_tiles.txt 2>&1
cp /tmp/pb_base.so $SO
