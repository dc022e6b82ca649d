export PYTHONPATH=$PWD
for v in 0 1; do
  echo "== SFV_GRAD_HOIST=$v"
  SFV_GRAD_HOIST=$v timeout 300 python scripts/microbench.py --config c2 --what jv --reps 200 2>&1 | grep -o '"jv_ms": [0-9.]*'
  SFV_GRAD_HOIST=$v timeout 300 python scripts/microbench.py --config c2 --what jv --reps 200 2>&1 | grep -o '"jv_ms": [0-9.]*'
done
SFV_GRAD_HOIST=1 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "jv or residual" 2>&1 | tail -2
