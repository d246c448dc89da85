#!/bin/bash
# 16-layer bench lines of one config per variant library
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
T=${RUN_TAG:-cfgb}
SO=paper_2312_05516_b200/libpensieve_b200.so
cp $SO /tmp/pb_base.so
for c in ${CFGS:-2}; do
for v in base ${VARIANTS}; do
  if [ "$v" = "base" ]; then cp /tmp/pb_base.so $SO; else cp paper_2312_05516_b200/variants/$v.so $SO; fi
  echo "== cfg$c $v $(timeout 300 python bench.py --config $c --steps 5 --warmup 3 --layers ${LAYERS:-16} --no-cpu-baseline --no-subconfigs 2>&1 | tail -1 | cut -c1-160)" >> gpurun_out/${T}_bench.txt
done
done
cp /tmp/pb_base.so $SO
