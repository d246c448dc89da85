cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
nvidia-smi > gpurun_out/b0_smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/b0_pytest.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/b0_cfg4.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline --layers 16 > gpurun_out/b0_cfg4_16.txt 2>&1
timeout 600 python bench.py --config 2 --no-cpu-baseline > gpurun_out/b0_cfg2.txt 2>&1
timeout 600 python bench.py --config 3 --no-cpu-baseline > gpurun_out/b0_cfg3.txt 2>&1
timeout 600 python scripts/shard_emulation.py > gpurun_out/b0_shard.txt 2>&1
