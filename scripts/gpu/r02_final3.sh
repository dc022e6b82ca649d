# Round-2 final evidence (fifth session: after the solo levels and the producer-side stage wait of the ILU sweep): tests, smoke, bench (both arms), configuration solves,
# J.v sweep, ncu launch list and --set full captures.
export PYTHONPATH=$PWD
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/r02_gpu.txt
lscpu | grep -E "Model name|^CPU\(s\)" >> gpurun_out/r02_gpu.txt
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02_pytest.log 2>&1; echo pytest=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/r02_bench.log 2>&1; echo bench=$?
timeout 900 python bench.py --impl reference --steps 32 --warmup 3 > gpurun_out/r02_bench_ref.log 2>&1; echo ref=$?
SFV_TIMING=1 timeout 1200 python scripts/run_configs.py --cases c1,c2,c3,c4 --out gpurun_out/r02_configs.json > gpurun_out/r02_configs.log 2>&1; echo configs=$?
timeout 1200 python scripts/jv_sweep.py --out gpurun_out/r02_jv_sweep.json > gpurun_out/r02_jv_sweep.log 2>&1; echo sweep=$?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --jfnk-steps 1 > gpurun_out/r02_ncu_launch.log 2>&1; echo launches=$?
for k in flux_pair_kernel grad_cell_kernel eps_perturb_kernel; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -s 3 -c 1 -o gpurun_out/r02_full_$k python scripts/microbench.py --what jv --reps 5 > gpurun_out/r02_ncu_$k.log 2>&1; echo $k=$?
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tri_stream_kernel -s 2 -c 2 -o gpurun_out/r02_full_tri_stream_kernel python scripts/microbench.py --what ilu --reps 4 > gpurun_out/r02_ncu_tri.log 2>&1; echo tri=$?
SFV_GMRES_GRAPH=0 timeout 600 ncu --set full --import-source on --clock-control none -k regex:arnoldi_kernel -s 10 -c 1 -o gpurun_out/r02_full_arnoldi_kernel python scripts/microbench.py --what gmres --reps 1 > gpurun_out/r02_ncu_arn.log 2>&1; echo arnoldi=$?
tail -3 gpurun_out/r02_pytest.log
