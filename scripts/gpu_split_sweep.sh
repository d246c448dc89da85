#!/bin/bash
# fused vs split launch timing (scripts/exp_fused_split.py) per variant library, N = 1, 8
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
T=${RUN_TAG:-split}
SO=paper_2312_05516_b200/libpensieve_b200.so
cp $SO /tmp/pb_base.so
for v in base ${VARIANTS}; do
  if [ "$v" = "base" ]; then cp /tmp/pb_base.so $SO; else cp paper_2312_05516_b200/variants/$v.so $SO; fi
  for wd in ${WORLDS:-1 8}; do echo "== $v $(timeout 300 python scripts/exp_fused_split.py ${CFG:-4} $wd 10 2>&1 | tail -1)" >> gpurun_out/${T}_split.txt; done
done
cp /tmp/pb_base.so $SO
