# Third session of round 2: re-verify the restored tree (tests, smoke, bench).
export PYTHONPATH=$PWD
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/r02c_pytest.log 2>&1; echo pytest=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02c_smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/r02c_bench.log 2>&1; echo bench=$?
tail -3 gpurun_out/r02c_pytest.log; tail -1 gpurun_out/r02c_bench.log
