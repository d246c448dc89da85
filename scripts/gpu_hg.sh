#!/bin/bash
# head-group decode check: quick hang probe, GPU attention/parity tests, fused split timings, benches
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
T=${RUN_TAG:-hg}
timeout 120 python scripts/exp_fused_split.py 4 1 3 > gpurun_out/${T}_probe.txt 2>&1 || { echo "probe failed rc=$?" >> gpurun_out/${T}_probe.txt; exit 0; }
timeout 1200 python -m pytest tests/test_attention_gpu.py tests/test_parity_full_gpu.py -x -q > gpurun_out/${T}_pytest.txt 2>&1
timeout 300 python scripts/exp_fused_split.py 2 1 10 > gpurun_out/${T}_split.txt 2>&1
timeout 300 python scripts/exp_fused_split.py 4 1 10 >> gpurun_out/${T}_split.txt 2>&1
for c in 4 2; do echo "== cfg$c $(timeout 300 python bench.py --config $c --steps 5 --warmup 3 --layers 16 --no-cpu-baseline --no-subconfigs 2>&1 | tail -1 | cut -c1-160)" >> gpurun_out/${T}_bench.txt; done
