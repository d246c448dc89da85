#!/bin/bash
# decode-path change: attention tests, per-CTA decode rate and 16-layer benches of configs 2/3
# against the previous build (variant "old"), alternating
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
T=${RUN_TAG:-dab}
SO=paper_2312_05516_b200/libpensieve_b200.so
timeout 900 python -m pytest tests/test_attention_gpu.py -x -q > gpurun_out/${T}_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/${T}_pytest.txt
cp $SO /tmp/pb_new.so
for v in new old; do cp /tmp/pb_new.so $SO; [ "$v" != "new" ] && cp paper_2312_05516_b200/variants/$v.so $SO; echo "== $v $(timeout 300 python scripts/exp_decode_per_sm.py 4096 2>&1 | tail -1)" >> gpurun_out/${T}_dec.txt; done
for r in 1 2 3; do
for v in new old; do
  cp /tmp/pb_new.so $SO; [ "$v" != "new" ] && cp paper_2312_05516_b200/variants/$v.so $SO
  for c in 2 3 4; do
    echo "== cfg$c $v $(timeout 300 python bench.py --config $c --steps 5 --warmup 3 --layers 16 --no-cpu-baseline --no-subconfigs 2>&1 | tail -1 | cut -c1-100)" >> gpurun_out/${T}_ab.txt
  done
done
done
cp /tmp/pb_new.so $SO
