#!/bin/bash
# quick check of a kernel change: GPU attention parity tests + tile bounds + short cfg4 bench
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
T=${RUN_TAG:-q}
timeout 900 python -m pytest tests/test_attention_gpu.py tests/test_parity_full_gpu.py -x -q > gpurun_out/${T}_pytest.txt 2>&1
timeout 300 python scripts/exp_tile_bounds.py > gpurun_out/${T}_bounds.txt 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --layers 16 --no-cpu-baseline --no-subconfigs > gpurun_out/${T}_bench.txt 2>&1
