export PYTHONPATH=$PWD
for v in "" divplain; do
  if [ -n "$v" ]; then export SFV_LIB=scripts/probes/variants/libsfv_$v.so; else unset SFV_LIB; fi
  echo "== variant ${v:-default}"
  timeout 300 python scripts/microbench.py --config c2 --what ilu --reps 20 2>&1 | grep -E "precond_apply" | sed 's/.*"precond_apply_ms_incl_sync"/apply_ms/' | head -3
done
unset SFV_LIB
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_golden.py tests/test_gpu_fullsize.py -q -k "ilu or sweep or golden or run_steps or lu_apply or transient" 2>&1 | tail -3
