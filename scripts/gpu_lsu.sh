#!/bin/bash
# decode V-on-LSU check: decode/attention tests, per-CTA decode rate, A/B benches
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
T=${RUN_TAG:-lsu}
timeout 120 python scripts/exp_decode_per_sm.py 4096 16 > gpurun_out/${T}_dec.txt 2>&1 || { echo "probe failed" >> gpurun_out/${T}_dec.txt; exit 0; }
timeout 1200 python -m pytest tests/test_attention_gpu.py tests/test_parity_full_gpu.py tests/test_edge_cases_gpu.py -x -q > gpurun_out/${T}_pytest.txt 2>&1
SO=paper_2312_05516_b200/libpensieve_b200.so
cp $SO /tmp/pb_base.so
cp paper_2312_05516_b200/variants/nolsu.so $SO
timeout 120 python scripts/exp_decode_per_sm.py 4096 16 >> gpurun_out/${T}_dec.txt 2>&1
cp /tmp/pb_base.so $SO
VARIANT=nolsu REPS=2 CFGS="2 4 3" RUN_TAG=$T bash scripts/gpu_ab.sh
