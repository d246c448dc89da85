#!/bin/bash
# decode-pipeline change check: GPU decode/attention tests, per-CTA decode rate, benches
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
T=${RUN_TAG:-dec}
timeout 1200 python -m pytest tests/test_attention_gpu.py tests/test_parity_full_gpu.py tests/test_swap_gpu.py -x -q > gpurun_out/${T}_pytest.txt 2>&1
timeout 300 python scripts/exp_decode_per_sm.py 4096 > gpurun_out/${T}_dec.txt 2>&1
for c in 3 2 4; do echo "== cfg$c $(timeout 300 python bench.py --config $c --steps 5 --warmup 3 --layers 16 --no-cpu-baseline --no-subconfigs 2>&1 | tail -1 | cut -c1-160)" >> gpurun_out/${T}_bench.txt; done
timeout 300 python scripts/exp_fused_split.py 2 1 10 > gpurun_out/${T}_split.txt 2>&1
timeout 300 python scripts/exp_fused_split.py 4 1 10 >> gpurun_out/${T}_split.txt 2>&1
