export PYTHONPATH=$PWD
for d in 0 1 0 1; do
SFV_EPS_DISCARD=$d timeout 300 python scripts/microbench.py --config c2 --what jv --reps 300 2>&1 | grep -o '"jv_ms": [0-9.]*' | sed "s/^/discard=$d /"
done
SFV_EPS_DISCARD=1 timeout 300 python bench.py --steps 20 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['value'], [ (s['kernel'], round(s['ms']*1e3,1)) for s in d['stages']])"
SFV_EPS_DISCARD=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "jv or residual or eps" 2>&1 | tail -2
