python -m pytest tests -m gpu -x -q > gpurun_out/final_pytest.log 2>&1; echo pytest=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo smoke=$?
python bench.py > gpurun_out/bench_final.log 2>&1; echo bench=$?
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_final.log 2>&1; echo ref=$?
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 2 --warmup 1 > gpurun_out/ncu_launch_final.log 2>&1; echo launches=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:flux_pair_kernel -s 4 -c 1 -o gpurun_out/prof_final_flux python scripts/microbench.py --what jv --reps 5 > gpurun_out/ncu_flux_final.log 2>&1; echo flux=$?
