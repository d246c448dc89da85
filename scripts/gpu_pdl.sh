#!/bin/bash
# PDL check: attention tests, shard emulation and 16-layer cfg4 bench, base vs variants
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
T=${RUN_TAG:-pdl}
SO=paper_2312_05516_b200/libpensieve_b200.so
cp $SO /tmp/pb_base.so
timeout 900 python -m pytest tests/test_attention_gpu.py tests/test_threads_gpu.py -x -q > gpurun_out/${T}_pytest.txt 2>&1
for v in base ${VARIANTS}; do
  if [ "$v" = "base" ]; then cp /tmp/pb_base.so $SO; else cp paper_2312_05516_b200/variants/$v.so $SO; fi
  echo "== $v $(timeout 600 python scripts/shard_emulation.py 2>&1 | tail -1)" >> gpurun_out/${T}_shard.txt
  echo "== $v $(timeout 300 python bench.py --steps 5 --warmup 3 --layers 16 --no-cpu-baseline --no-subconfigs 2>&1 | tail -1 | cut -c1-120)" >> gpurun_out/${T}_bench.txt
done
cp /tmp/pb_base.so $SO
