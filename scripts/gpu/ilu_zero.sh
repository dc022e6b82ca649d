export PYTHONPATH=$PWD
for i in 1 2 3; do
  timeout 300 python scripts/microbench.py --config c2 --what ilu --reps 60 2>&1 | grep -o '"precond_apply_ms_incl_sync": [0-9.]*'
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_golden.py tests/test_gpu_fullsize.py -q -x -k "ilu or sweep or golden or precond or sequential_reductions_bit" 2>&1 | tail -2
