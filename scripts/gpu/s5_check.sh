# Session-5 check after the coupled (oblique symmetry) preconditioner: GPU tests, smoke, both bench arms.
export PYTHONPATH=$PWD
( time timeout 1700 python -m pytest tests -m gpu -q ) > gpurun_out/s5_pytest.log 2>&1; echo pytest=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s5_smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/s5_bench.log 2>&1; echo bench=$?
timeout 900 python bench.py --impl reference --steps 32 --warmup 3 > gpurun_out/s5_bench_ref.log 2>&1; echo ref=$?
tail -3 gpurun_out/s5_pytest.log; tail -n 1 gpurun_out/s5_bench.log | cut -c1-600; tail -n 1 gpurun_out/s5_bench_ref.log | cut -c1-900
