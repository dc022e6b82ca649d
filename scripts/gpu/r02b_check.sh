export PYTHONPATH=$PWD
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -5
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r02b.json 2> gpurun_out/bench_r02b.err; echo bench=$?
tail -c 1500 gpurun_out/bench_r02b.json
