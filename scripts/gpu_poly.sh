#!/bin/bash
# exp2 offload ratios: config-4 tile bounds and 16-layer benches, base vs variants
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
T=${RUN_TAG:-poly}
SO=paper_2312_05516_b200/libpensieve_b200.so
cp $SO /tmp/pb_base.so
for r in 1 2; do
for v in base ${VARIANTS}; do
  cp /tmp/pb_base.so $SO; [ "$v" != "base" ] && cp paper_2312_05516_b200/variants/$v.so $SO
  echo "== $v $(timeout 300 python scripts/exp_tile_bounds.py 10 16 2>&1 | tail -1 | cut -c1-70) $(timeout 300 python bench.py --config 4 --steps 5 --warmup 3 --layers 16 --no-cpu-baseline --no-subconfigs 2>&1 | tail -1 | cut -c1-80)" >> gpurun_out/${T}.txt
done
done
cp /tmp/pb_base.so $SO
