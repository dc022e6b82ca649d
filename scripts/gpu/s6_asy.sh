# Session 6: Hooke face pass with every operand staged by cp.async one tile ahead
export PYTHONPATH=$PWD
for v in "" asy4 asy3 "" asy4 asy3; do
  if [ -n "$v" ]; then export SFV_LIB=scripts/probes/variants/libsfv_$v.so; else unset SFV_LIB; fi
  for c in c2 c4; do
  timeout 300 python scripts/microbench.py --config $c --what jv --reps 300 2>&1 | grep -o '"jv_ms": [0-9.]*' | sed "s/^/${v:-default} $c /"
  done
done
for v in asy4 asy3; do
export SFV_LIB=scripts/probes/variants/libsfv_$v.so
timeout 900 python -m pytest tests -m gpu -q -x -k "jv or residual or golden or fullsize or known or tet or host_buffers or transient" 2>&1 | tail -4
done
