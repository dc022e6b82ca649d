export PYTHONPATH=$PWD
timeout 300 python scripts/microbench.py --config c2 --what ilu --reps 40 2>&1 | grep -o '"precond_apply_ms_incl_sync": [0-9.]*'
timeout 300 python scripts/microbench.py --config c2 --what ilu --reps 40 2>&1 | grep -o '"precond_apply_ms_incl_sync": [0-9.]*'
SFV_HOST_PRECOND=1 timeout 300 python scripts/microbench.py --config c2 --what ilu --reps 40 2>&1 | grep -o '"precond_apply_ms_incl_sync": [0-9.]*'
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_golden.py -q -x -k "ilu or sweep or golden or precond" 2>&1 | tail -2
SFV_TIMING=1 timeout 600 python scripts/run_configs.py --cases c2 2>&1 | grep -E '"case"|gmres [0-9]+ iters' | cut -c1-300
