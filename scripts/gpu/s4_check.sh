# Session-4 sanity: GPU tests, smoke, bench (both arms) on the restored checkpoint.
export PYTHONPATH=$PWD
( time timeout 1700 python -m pytest tests -m gpu -q ) > gpurun_out/s4_pytest.log 2>&1; echo pytest=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4_smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/s4_bench.log 2>&1; echo bench=$?
tail -3 gpurun_out/s4_pytest.log; tail -2 gpurun_out/s4_bench.log
