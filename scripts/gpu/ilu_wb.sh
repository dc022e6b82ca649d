export PYTHONPATH=$PWD
for v in "" wb0 "" wb0; do
  if [ -n "$v" ]; then export SFV_LIB=scripts/probes/variants/libsfv_$v.so; else unset SFV_LIB; fi
  timeout 300 python scripts/microbench.py --config c2 --what ilu --reps 60 2>&1 | grep -o '"precond_apply_ms_incl_sync": [0-9.]*' | sed "s/^/${v:-wb1} /"
done
unset SFV_LIB
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_golden.py tests/test_gpu_fullsize.py -q -x -k "ilu or sweep or golden or precond or sequential_reductions_bit" 2>&1 | tail -2
SFV_TIMING=1 timeout 900 python scripts/run_configs.py --cases c2,c4 2>&1 | grep -o '"case": "c[24]".*"krylov_total": [0-9]*' | cut -c1-200
