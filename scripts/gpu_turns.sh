#!/bin/bash
# exponential turns: smoke under a short timeout, tile trace, tile bounds (new / noturn / old)
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
T=${RUN_TAG:-tu}
SO=paper_2312_05516_b200/libpensieve_b200.so
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.txt 2>&1
rc=$?; echo "smoke rc=$rc" >> gpurun_out/${T}_smoke.txt
[ $rc -ne 0 ] && exit 0
cp $SO /tmp/pb_new.so
cp paper_2312_05516_b200/variants/tt.so $SO
echo "== tt $(timeout 300 python scripts/trace_tiles.py 4 2>&1 | tail -1 | cut -c1-700)" >> gpurun_out/${T}_trace.txt
for v in new ${VARIANTS}; do
  cp /tmp/pb_new.so $SO; [ "$v" != "new" ] && cp paper_2312_05516_b200/variants/$v.so $SO
  echo "== $v $(timeout 300 python scripts/exp_tile_bounds.py 10 16 2>&1 | tail -1 | cut -c1-90)" >> gpurun_out/${T}_bounds.txt
done
cp /tmp/pb_new.so $SO
for c in 4 2 3; do
for v in new old; do
  cp /tmp/pb_new.so $SO; [ "$v" != "new" ] && cp paper_2312_05516_b200/variants/$v.so $SO
  echo "== cfg$c $v $(timeout 300 python bench.py --config $c --steps 5 --warmup 3 --layers 16 --no-cpu-baseline --no-subconfigs 2>&1 | tail -1 | cut -c1-100)" >> gpurun_out/${T}_ab.txt
done
done
cp /tmp/pb_new.so $SO
