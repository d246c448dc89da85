#!/bin/bash
# Quick perf + correctness pass (no ncu): probes, then bench lines for configs 4, 2, 3.
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
T=${RUN_TAG:-quick}
for c in ${CASES:-p1 p5 mix d3 cfg2 cfg3 cfg4}; do
  timeout 60 python scripts/debug_attn.py $c >> gpurun_out/${T}_probe.txt 2>&1 || echo "$c: rc=$?" >> gpurun_out/${T}_probe.txt
done
for cfg in ${CFGS:-4 2 3}; do
  timeout 600 python bench.py --config $cfg --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/${T}_bench_cfg$cfg.txt 2>&1
done
