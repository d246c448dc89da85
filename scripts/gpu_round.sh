#!/bin/bash
# Round evidence pass: GPU tests + smoke, then the profile pass (bench lines, launch lists, ncu).
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
T=${RUN_TAG:-round}
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -30 > gpurun_out/${T}_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.txt 2>&1
timeout 600 python bench.py --config 5 > gpurun_out/${T}_bench_cfg5.txt 2>&1
RUN_TAG=$T bash scripts/gpu_profile.sh
