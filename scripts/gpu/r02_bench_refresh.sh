export PYTHONPATH=$PWD
timeout 900 python bench.py > gpurun_out/r02_bench.log 2>&1; echo bench=$?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --jfnk-steps 1 > gpurun_out/r02_ncu_launch.log 2>&1; echo launches=$?
tail -c 600 gpurun_out/r02_bench.log
