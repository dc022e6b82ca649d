# Round-2 evidence refresh after the ILU sweep changes: tests, smoke, bench, configuration solves,
# launch list, ILU sweep capture.
export PYTHONPATH=$PWD
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02_pytest.log 2>&1; echo pytest=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/r02_bench.log 2>&1; echo bench=$?
SFV_TIMING=1 timeout 1200 python scripts/run_configs.py --cases c1,c2,c3,c4 --out gpurun_out/r02_configs.json > gpurun_out/r02_configs.log 2>&1; echo configs=$?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --jfnk-steps 1 > gpurun_out/r02_ncu_launch.log 2>&1; echo launches=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tri_stream_kernel -s 2 -c 2 -o gpurun_out/r02_full_tri_stream_kernel python scripts/microbench.py --what ilu --reps 4 > gpurun_out/r02_ncu_tri.log 2>&1; echo tri=$?
tail -3 gpurun_out/r02_pytest.log
