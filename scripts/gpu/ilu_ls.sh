export PYTHONPATH=$PWD
for v in "" pw0 "" pw0; do
  if [ -n "$v" ]; then export SFV_LIB=scripts/probes/variants/libsfv_$v.so; else unset SFV_LIB; fi
  timeout 300 python scripts/microbench.py --config c2 --what ilu --reps 60 2>&1 | grep -o '"precond_apply_ms_incl_sync": [0-9.]*' | sed "s/^/${v:-pwait} /"
done
unset SFV_LIB
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_golden.py -q -x -k "ilu or sweep or golden or precond" 2>&1 | tail -2
