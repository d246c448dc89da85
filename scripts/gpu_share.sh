#!/bin/bash
# decode CTA share at >= 25% decode (configs 2 and 5): base vs variants, alternating
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
T=${RUN_TAG:-share}
SO=paper_2312_05516_b200/libpensieve_b200.so
cp $SO /tmp/pb_base.so
for r in 1 2; do
for v in base ${VARIANTS}; do
  cp /tmp/pb_base.so $SO; [ "$v" != "base" ] && cp paper_2312_05516_b200/variants/$v.so $SO
  for c in 2 5; do
    echo "== cfg$c $v $(timeout 300 python bench.py --config $c --steps 5 --warmup 3 --layers 16 --no-cpu-baseline --no-subconfigs 2>&1 | tail -1 | cut -c1-90)" >> gpurun_out/${T}.txt
  done
done
done
cp /tmp/pb_base.so $SO
