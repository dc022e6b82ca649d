set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
lscpu | grep -E "Model name|^CPU\(s\)|Thread"
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
SFV_TIMING=1 timeout 600 python scripts/run_configs.py --cases c2 > gpurun_out/r02_base_c2.log 2>&1
tail -5 gpurun_out/r02_base_c2.log
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu > gpurun_out/r02_base_bench.json 2> gpurun_out/r02_base_bench.err
cat gpurun_out/r02_base_bench.json | head -c 3000
