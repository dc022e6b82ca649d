export PYTHONPATH=$PWD
for v in "" wgk0 "" wgk0; do
  if [ -n "$v" ]; then export SFV_LIB=scripts/probes/variants/libsfv_$v.so; else unset SFV_LIB; fi
  timeout 300 python scripts/microbench.py --config c2 --what jv --reps 300 2>&1 | grep -o '"jv_ms": [0-9.]*' | sed "s/^/${v:-keep} /"
done
export SFV_LIB=scripts/probes/variants/libsfv_wgk0.so
SFV_GMRES_GRAPH=0 SFV_TIMING=1 timeout 300 python scripts/microbench.py --config c2 --what gmres --reps 1 2>&1 | grep -E "gmres [0-9]+ iters" | cut -c1-120
unset SFV_LIB
SFV_GMRES_GRAPH=0 SFV_TIMING=1 timeout 300 python scripts/microbench.py --config c2 --what gmres --reps 1 2>&1 | grep -E "gmres [0-9]+ iters" | cut -c1-120
