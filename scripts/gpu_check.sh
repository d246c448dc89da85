#!/bin/bash
# GPU bring-up: per-case probes (each under its own timeout), then the GPU test suite.
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
OUT=gpurun_out/${RUN_TAG:-run}
for c in ${CASES:-p1 p2 p3 p4 p5 p6 d1 d2 d3 d4 mix cfg2 cfg3 cfg4}; do
  timeout 60 python scripts/debug_attn.py $c >> ${OUT}_probe.txt 2>&1 || echo "$c: rc=$?" >> ${OUT}_probe.txt
done
if [ -z "$NO_PYTEST" ]; then
  timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -40 > ${OUT}_pytest.txt
fi
if [ -n "$BENCH" ]; then
  timeout 600 python bench.py $BENCH > ${OUT}_bench.txt 2>&1
fi
