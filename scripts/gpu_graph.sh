#!/bin/bash
# graph-launched layer loop: new tests, attention tests, bench line, shard emulation
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
T=${RUN_TAG:-gr}
timeout 900 python -m pytest tests/test_run_layers_gpu.py tests/test_attention_gpu.py tests/test_soak_gpu.py -x -q > gpurun_out/${T}_pytest.txt 2>&1
timeout 300 python scripts/exp_graph.py > gpurun_out/${T}_graph.txt 2>&1
timeout 600 python bench.py > gpurun_out/${T}_bench.txt 2>&1
timeout 300 python scripts/shard_emulation.py > gpurun_out/${T}_shard.txt 2>&1
