#!/bin/bash
# tile-bounds experiment (config-4 prefill tiles alone) for the product library and variants
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
T=${RUN_TAG:-bounds}
SO=paper_2312_05516_b200/libpensieve_b200.so
cp $SO /tmp/pb_base.so
for v in base ${VARIANTS}; do
  if [ "$v" = "base" ]; then cp /tmp/pb_base.so $SO; else cp paper_2312_05516_b200/variants/$v.so $SO; fi
  echo "== $v $(timeout 300 python scripts/exp_tile_bounds.py ${REPS:-10} ${CHUNKS:-16} 2>&1 | tail -1)" >> gpurun_out/${T}_bounds.txt
done
cp /tmp/pb_base.so $SO
