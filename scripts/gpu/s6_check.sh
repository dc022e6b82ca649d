# Session-6 re-validation on the restored checkpoint: GPU tests, smoke, both bench arms.
export PYTHONPATH=$PWD
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/s6_gpu.txt
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/s6_pytest.log 2>&1; echo pytest=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s6_smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/s6_bench.log 2>&1; echo bench=$?
timeout 900 python bench.py --impl reference --steps 32 --warmup 3 > gpurun_out/s6_bench_ref.log 2>&1; echo ref=$?
tail -3 gpurun_out/s6_pytest.log; tail -1 gpurun_out/s6_bench.log | cut -c1-1500
