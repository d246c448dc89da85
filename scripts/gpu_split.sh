#!/bin/bash
# kv-split tile items (small shards): smoke, the attention / parity / edge / soak tests, shard
# emulation of this build and of the previous one (variant "old"), alternating
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
T=${RUN_TAG:-sp}
SO=paper_2312_05516_b200/libpensieve_b200.so
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.txt 2>&1
rc=$?; echo "smoke rc=$rc" >> gpurun_out/${T}_smoke.txt
[ $rc -ne 0 ] && exit 0
cp $SO /tmp/pb_new.so
for r in 1 2; do
for v in new old; do
  cp /tmp/pb_new.so $SO; [ "$v" != "new" ] && cp paper_2312_05516_b200/variants/$v.so $SO
  echo "== $v $(timeout 300 python scripts/shard_emulation.py 2>&1 | tail -1)" >> gpurun_out/${T}_shard.txt
done
done
cp /tmp/pb_new.so $SO
timeout 1500 python -m pytest tests/test_attention_gpu.py tests/test_parity_full_gpu.py tests/test_edge_cases_gpu.py tests/test_soak_gpu.py tests/test_run_layers_gpu.py -x -q > gpurun_out/${T}_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/${T}_pytest.txt
