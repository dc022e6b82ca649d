# J.v epilogue quotient by reciprocal + Markstein correction (SFV_JV_DIV_CORR): timing and bitwise check
export PYTHONPATH=$PWD
for c in c2 c4 c3; do
for lib in "" scripts/probes/variants/libsfv_divc.so; do
  for r in 1 2; do
  SFV_LIB=$lib timeout 300 python scripts/microbench.py --config $c --what jv --reps 400 2>&1 | grep -o '"jv_ms": [0-9.]*' | sed "s|^|$c ${lib:-default} |"
  done
done
done
SFV_LIB=scripts/probes/variants/libsfv_divc.so timeout 900 python -m pytest -q -x tests/test_gpu_fullsize.py -k "bitwise or reference_eps" tests/test_gpu_parity.py 2>&1 | tail -3
