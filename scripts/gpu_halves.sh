#!/bin/bash
# column-half softmax warpgroups: correctness first (attention tests under a timeout), then
# tile bounds and 16-layer benches against the previous kernel (variant "old")
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
T=${RUN_TAG:-hv}
SO=paper_2312_05516_b200/libpensieve_b200.so
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.txt 2>&1
rc=$?; echo "smoke rc=$rc" >> gpurun_out/${T}_smoke.txt
[ $rc -ne 0 ] && exit 0
timeout 900 python -m pytest tests/test_attention_gpu.py -x -q > gpurun_out/${T}_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/${T}_pytest.txt
cp $SO /tmp/pb_new.so
for v in new old; do
  cp paper_2312_05516_b200/variants/old.so $SO; [ "$v" = "new" ] && cp /tmp/pb_new.so $SO
  echo "== $v $(timeout 300 python scripts/exp_tile_bounds.py 10 16 2>&1 | tail -1)" >> gpurun_out/${T}_bounds.txt
done
for r in 1 2; do
for c in 4 2; do
for v in new old; do
  cp paper_2312_05516_b200/variants/old.so $SO; [ "$v" = "new" ] && cp /tmp/pb_new.so $SO
  echo "== cfg$c $v $(timeout 300 python bench.py --config $c --steps 5 --warmup 3 --layers 16 --no-cpu-baseline --no-subconfigs 2>&1 | tail -1 | cut -c1-110)" >> gpurun_out/${T}_ab.txt
done
done
done
cp /tmp/pb_new.so $SO
