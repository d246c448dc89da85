#!/bin/bash
# Round evidence pass: GPU tests, smoke, bench lines for every config (+ reference arm),
# ncu launch lists and one full ncu capture per hot kernel, a 1-rank torchrun bench.
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
T=${RUN_TAG:-final}
nproc > gpurun_out/${T}_nproc.txt
timeout 600 python -m pytest tests -m gpu -q > gpurun_out/${T}_pytest.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/${T}_bench_cfg4.txt 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${T}_bench_reference.txt 2>&1
for c in 2 3; do timeout 600 python bench.py --config $c > gpurun_out/${T}_bench_cfg$c.txt 2>&1; done
timeout 600 python bench.py --config 5 > gpurun_out/${T}_bench_cfg5.txt 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 1 --steps 3 --warmup 3 --layers 8 --no-cpu-baseline > gpurun_out/${T}_torchrun1.txt 2>&1
timeout 300 python scripts/shard_emulation.py > gpurun_out/${T}_shard.txt 2>&1
timeout 600 python scripts/bench_strawmen.py --contexts 256,1024,4096 --reps 10 --out gpurun_out/${T}_strawmen.json > gpurun_out/${T}_strawmen.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:attn -c 40 --csv \
  --log-file gpurun_out/${T}_launches_cfg4.csv python bench.py --steps 1 --warmup 3 --layers 8 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:attn -c 40 --csv \
  --log-file gpurun_out/${T}_launches_cfg3.csv python bench.py --config 3 --steps 1 --warmup 3 --layers 8 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fused -s 2 -c 1 \
  -o gpurun_out/${T}_fused python bench.py --steps 1 --warmup 3 --layers 2 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_decode -s 2 -c 1 \
  -o gpurun_out/${T}_decode python bench.py --config 3 --steps 1 --warmup 3 --layers 2 --no-cpu-baseline > /dev/null 2>&1
