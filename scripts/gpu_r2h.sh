#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
T=${RUN_TAG:-r2h}
SO=paper_2312_05516_b200/libpensieve_b200.so
cp $SO /tmp/pb_base.so
for v in ${VARIANTS:-tt ttp4 tta2}; do
  cp paper_2312_05516_b200/variants/$v.so $SO
  echo "== $v" >> gpurun_out/${T}_trace.txt
  timeout 300 python scripts/trace_tiles.py 4 >> gpurun_out/${T}_trace.txt 2>&1
done
cp /tmp/pb_base.so $SO
