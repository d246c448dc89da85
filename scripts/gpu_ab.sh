#!/bin/bash
# A/B: 16-layer benches of configs ${CFGS} alternating base and one variant, ${REPS} rounds
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
T=${RUN_TAG:-ab}
SO=paper_2312_05516_b200/libpensieve_b200.so
cp $SO /tmp/pb_base.so
for r in $(seq 1 ${REPS:-2}); do
for c in ${CFGS:-4 2}; do
for v in base ${VARIANT}; do
  if [ "$v" = "base" ]; then cp /tmp/pb_base.so $SO; else cp paper_2312_05516_b200/variants/$v.so $SO; fi
  echo "== cfg$c $v $(timeout 300 python bench.py --config $c --steps 5 --warmup 3 --layers ${LAYERS:-16} --no-cpu-baseline --no-subconfigs 2>&1 | tail -1 | cut -c1-110)" >> gpurun_out/${T}_ab.txt
done
done
done
cp /tmp/pb_base.so $SO
