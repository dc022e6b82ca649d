export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "host_buffers" 2>&1 | tail -2
for c in 4 8 16 8 16 4; do
SFV_JV_HOST_CHUNKS=$c timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-jfnk 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('chunks=$c', round(d['value']), round(d['e2e']['value'],1))"
done
