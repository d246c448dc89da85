#!/bin/bash
# Variant sweep (profiling experiments, never the product): each prebuilt variant library
# (scripts/build_variants.sh -> paper_2312_05516_b200/variants/<name>.so) is copied over the
# product library of this box's scratch copy, then probed for parity and timed on a short
# bench.  VARIANTS="name ..." ("base" = the product library as shipped).
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
T=${RUN_TAG:-var}
SO=paper_2312_05516_b200/libpensieve_b200.so
cp $SO /tmp/pb_base.so
if [ -n "$PYTEST" ]; then timeout 900 python -m pytest $PYTEST -x -q 2>&1 | tail -15 > gpurun_out/${T}_pytest.txt; fi
for v in ${VARIANTS}; do
  if [ "$v" = "base" ]; then cp /tmp/pb_base.so $SO; else cp paper_2312_05516_b200/variants/$v.so $SO; fi
  echo "== $v" >> gpurun_out/${T}_probe.txt
  timeout 120 python scripts/debug_attn.py ${PROBE:-cfg4} >> gpurun_out/${T}_probe.txt 2>&1
  timeout 300 python bench.py --config ${CFG:-4} --steps 5 --warmup 3 --layers ${LAYERS:-16} --no-cpu-baseline > gpurun_out/${T}_$v.txt 2>&1
done
cp /tmp/pb_base.so $SO
