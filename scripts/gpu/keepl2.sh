export PYTHONPATH=$PWD
for v in "" kl0 "" kl0; do
  if [ -n "$v" ]; then export SFV_LIB=scripts/probes/variants/libsfv_$v.so; else unset SFV_LIB; fi
  timeout 300 python scripts/microbench.py --config c2 --what jv --reps 300 2>&1 | grep -o '"jv_ms": [0-9.]*' | sed "s/^/${v:-keepl2} /"
done
unset SFV_LIB
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-jfnk 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['value'], [ (s['kernel'], round(s['ms']*1e3,1)) for s in d['stages']])"
SFV_GMRES_GRAPH=0 SFV_TIMING=1 timeout 300 python scripts/microbench.py --config c2 --what gmres --reps 1 2>&1 | grep -E "gmres [0-9]+ iters" | cut -c1-120
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "jv or eps" 2>&1 | tail -2
