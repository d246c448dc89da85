#!/bin/bash
# kernel change check: all GPU attention tests + 16-layer benches of configs 4, 2, 3, 5
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
T=${RUN_TAG:-allcfg}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest.txt 2>&1
for c in 4 2 3 5; do echo "== cfg$c $(timeout 300 python bench.py --config $c --steps 5 --warmup 3 --layers 16 --no-cpu-baseline --no-subconfigs 2>&1 | tail -1 | cut -c1-160)" >> gpurun_out/${T}_bench.txt; done
