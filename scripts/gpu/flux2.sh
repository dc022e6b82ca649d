export PYTHONPATH=$PWD
for v in "" f2c8 f2c12; do
  if [ -n "$v" ]; then export SFV_LIB=scripts/probes/variants/libsfv_$v.so; else unset SFV_LIB; fi
  for f in 0 1; do
    SFV_FLUX2=$f timeout 300 python scripts/microbench.py --config c2 --what jv --reps 300 2>&1 | grep -o '"jv_ms": [0-9.]*' | sed "s/^/${v:-c10} flux2=$f /"
  done
done
unset SFV_LIB
SFV_FLUX2=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "jv or residual" 2>&1 | tail -2
