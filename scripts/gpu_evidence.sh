#!/bin/bash
# Round evidence pass: all GPU tests, smoke, the default bench line (cfg4 + cfg2/3/5
# sub-results) and the reference arm, shard emulation, 1-rank torchrun, ncu launch list and
# full captures of the fused kernel (cfg4) and the decode kernel (cfg3).
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
T=${RUN_TAG:-ev}
nproc > gpurun_out/${T}_nproc.txt
timeout 1500 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/${T}_pytest.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/${T}_bench.txt 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${T}_bench_ref.txt 2>&1
timeout 600 python scripts/shard_emulation.py > gpurun_out/${T}_shard.txt 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 1 --steps 3 --warmup 3 --layers 8 --no-cpu-baseline --no-subconfigs > gpurun_out/${T}_torchrun1.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:attn -c 40 --csv \
  --log-file gpurun_out/${T}_launches_cfg4.csv python bench.py --steps 1 --warmup 3 --layers 8 --no-cpu-baseline --no-subconfigs > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fused -s 2 -c 1 \
  -o gpurun_out/${T}_fused python bench.py --steps 1 --warmup 3 --layers 2 --no-cpu-baseline --no-subconfigs > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_decode -s 2 -c 1 \
  -o gpurun_out/${T}_decode python bench.py --config 3 --steps 1 --warmup 3 --layers 2 --no-cpu-baseline --no-subconfigs > /dev/null 2>&1
