#!/bin/bash
# kernel change check: attention parity tests, tile bounds + 16-layer bench for the product
# library vs variants, per-tile trace (tt), full default bench line.
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
T=${RUN_TAG:-r2k}
SO=paper_2312_05516_b200/libpensieve_b200.so
cp $SO /tmp/pb_base.so
timeout 900 python -m pytest tests/test_attention_gpu.py tests/test_parity_full_gpu.py -x -q > gpurun_out/${T}_pytest.txt 2>&1
for v in base ${VARIANTS}; do
  if [ "$v" = "base" ]; then cp /tmp/pb_base.so $SO; else cp paper_2312_05516_b200/variants/$v.so $SO; fi
  echo "== $v $(timeout 300 python scripts/exp_tile_bounds.py 10 2>&1 | tail -1)" >> gpurun_out/${T}_bounds.txt
  echo "== $v $(timeout 300 python bench.py --steps 5 --warmup 3 --layers 16 --no-cpu-baseline --no-subconfigs 2>&1 | tail -1)" >> gpurun_out/${T}_bench16.txt
done
if [ -f paper_2312_05516_b200/variants/tt.so ]; then
  cp paper_2312_05516_b200/variants/tt.so $SO
  timeout 300 python scripts/trace_tiles.py 4 > gpurun_out/${T}_trace.txt 2>&1
fi
cp /tmp/pb_base.so $SO
[ -n "$FULL" ] && timeout 900 python bench.py --no-cpu-baseline > gpurun_out/${T}_bench.txt 2>&1
true
