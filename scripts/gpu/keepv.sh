export PYTHONPATH=$PWD
for k in 1 0 1 0; do
SFV_EPS_KEEPV=$k timeout 300 python scripts/microbench.py --config c2 --what jv --reps 300 2>&1 | grep -o '"jv_ms": [0-9.]*' | sed "s/^/keepv=$k /"
done
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-jfnk 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['value'], [ (s['kernel'], round(s['ms']*1e3,1)) for s in d['stages']])"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_known_answers.py -q -x -k "jv or eps or residual or graph or gmres" 2>&1 | tail -2
