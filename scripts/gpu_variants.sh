#!/bin/bash
# Variant sweep (profiling experiments): for each prebuilt variant library, a cfg4 parity probe
# and a short cfg4 bench; then PB_ABLATE runs.  VARIANTS="name.so ..." ("" = product library).
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
T=${RUN_TAG:-var}
if [ -n "$PYTEST" ]; then timeout 900 python -m pytest $PYTEST -x -q 2>&1 | tail -15 > gpurun_out/${T}_pytest.txt; fi
for v in ${VARIANTS}; do
  lib=$v; [ "$v" = "base" ] && lib=""
  echo "== $v" >> gpurun_out/${T}_probe.txt
  PB_LIB=$lib timeout 120 python scripts/debug_attn.py ${PROBE:-cfg4} >> gpurun_out/${T}_probe.txt 2>&1
  PB_ONLY=${ONLY:-0} PB_LIB=$lib timeout 300 python bench.py --config ${CFG:-4} --steps 5 --warmup 3 --layers 16 --no-cpu-baseline > gpurun_out/${T}_$v.txt 2>&1
done
for a in ${EXTRA}; do  # "name:ENV=VAL,ENV2=VAL" bench runs of the product library
  kv=${a#*:}
  env ${kv//,/ } timeout 300 python bench.py --config ${CFG:-4} --steps 5 --warmup 3 --layers 16 --no-cpu-baseline > gpurun_out/${T}_x_${a%%:*}.txt 2>&1
done
for a in ${ABLATE}; do
  PB_ABLATE=${a#*:} PB_LIB=${a%%:*} timeout 300 python bench.py --config ${CFG:-4} --steps 5 --warmup 3 --layers 16 --no-cpu-baseline > gpurun_out/${T}_ablate_${a/:/_}.txt 2>&1
done
