#!/bin/bash
# tile-pipeline bounds: page size sweep x {product, no-softmax, no-exp2} builds
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
T=${RUN_TAG:-r2d}
SO=paper_2312_05516_b200/libpensieve_b200.so
cp $SO /tmp/pb_base.so
for v in base a1 a2; do
  if [ "$v" = "base" ]; then cp /tmp/pb_base.so $SO; else cp paper_2312_05516_b200/variants/$v.so $SO; fi
  echo "== $v" >> gpurun_out/${T}_bounds.txt
  timeout 300 python scripts/exp_tile_bounds.py >> gpurun_out/${T}_bounds.txt 2>&1
done
cp /tmp/pb_base.so $SO
