#!/bin/bash
# Round-2 check: GPU tests (incl. full-length parity, swap hazards, threads), smoke, the
# default bench line (cfg4 + cfg2/3/5 sub-results), the reference arm.
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
T=${RUN_TAG:-r2a}
nproc > gpurun_out/${T}_nproc.txt
timeout 1500 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/${T}_pytest.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/${T}_bench.txt 2>&1
timeout 600 python bench.py --impl reference > gpurun_out/${T}_bench_ref.txt 2>&1
