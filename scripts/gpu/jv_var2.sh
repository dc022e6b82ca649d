export PYTHONPATH=$PWD
for lib in "" scripts/probes/variants/libsfv_gminb3.so scripts/probes/variants/libsfv_gminb2.so; do
  echo "== lib ${lib:-default}"
  for h in 0 1; do
    SFV_LIB=$lib SFV_GRAD_HOIST=$h timeout 300 python scripts/microbench.py --config c2 --what jv --reps 300 2>&1 | grep -o '"jv_ms": [0-9.]*' | sed "s/^/hoist=$h /"
  done
done
for c in c3 c4; do
  for h in 0 1; do
    SFV_GRAD_HOIST=$h timeout 300 python scripts/microbench.py --config $c --what jv --reps 200 2>&1 | grep -o '"jv_ms": [0-9.]*' | sed "s/^/$c hoist=$h /"
  done
done
