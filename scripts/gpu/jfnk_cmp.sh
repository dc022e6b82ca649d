export PYTHONPATH=$PWD
SFV_TIMING=1 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu 2> gpurun_out/jc_bench.err | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('bench jfnk', d['jfnk']['solve_seconds'])"
grep "gmres\|device ilu\|ilu sweep" gpurun_out/jc_bench.err | tail -4
SFV_TIMING=1 timeout 600 python scripts/run_configs.py --cases c2 2> gpurun_out/jc_cfg.err | grep -o '"solve_seconds": [0-9.]*'
grep "gmres\|ilu sweep" gpurun_out/jc_cfg.err | tail -3
SFV_TIMING=1 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --jfnk-steps 1 2> gpurun_out/jc_bench2.err | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('bench jfnk 2', d['jfnk']['solve_seconds'])"
