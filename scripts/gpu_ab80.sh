#!/bin/bash
# A/B at the full 80-layer config-4 step (the power-capped regime): base vs ${VARIANT},
# ${REPS} alternating rounds; prints value and median SM clock of each run
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
T=${RUN_TAG:-ab80}
SO=paper_2312_05516_b200/libpensieve_b200.so
cp $SO /tmp/pb_base.so
for r in $(seq 1 ${REPS:-3}); do
for v in base ${VARIANT}; do
  if [ "$v" = "base" ]; then cp /tmp/pb_base.so $SO; else cp paper_2312_05516_b200/variants/$v.so $SO; fi
  timeout 300 python bench.py --no-cpu-baseline --no-subconfigs ${ARGS} 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); c=d.get('clocks',{})
print('$v', round(d['value'],1), d['ms_per_step'], c.get('sm_mhz'), c.get('reasons'))" >> gpurun_out/${T}.txt 2>&1
done
done
cp /tmp/pb_base.so $SO
