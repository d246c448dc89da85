#!/bin/bash
# decode ring-depth A/B: per-CTA decode rate and 16-layer benches for base and each variant
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
T=${RUN_TAG:-stg}
SO=paper_2312_05516_b200/libpensieve_b200.so
cp $SO /tmp/pb_base.so
for v in base ${VARIANTS}; do
  if [ "$v" = "base" ]; then cp /tmp/pb_base.so $SO; else cp paper_2312_05516_b200/variants/$v.so $SO; fi
  echo "== $v" >> gpurun_out/${T}_dec.txt
  timeout 300 python scripts/exp_decode_per_sm.py 4096 >> gpurun_out/${T}_dec.txt 2>&1
  timeout 600 python -m pytest tests/test_attention_gpu.py -x -q 2>&1 | tail -2 >> gpurun_out/${T}_dec.txt
done
for r in 1 2; do
for c in 3 2 4; do
for v in base ${VARIANTS}; do
  if [ "$v" = "base" ]; then cp /tmp/pb_base.so $SO; else cp paper_2312_05516_b200/variants/$v.so $SO; fi
  echo "== cfg$c $v $(timeout 300 python bench.py --config $c --steps 5 --warmup 3 --layers 16 --no-cpu-baseline --no-subconfigs 2>&1 | tail -1 | cut -c1-110)" >> gpurun_out/${T}_ab.txt
done
done
done
cp /tmp/pb_base.so $SO
