export PYTHONPATH=$PWD
for pf in 1 0 1 0; do
SFV_ARN_PF=$pf SFV_GMRES_GRAPH=0 SFV_TIMING=1 timeout 300 python scripts/microbench.py --config c2 --what gmres --reps 1 2>&1 | grep -E "gmres [0-9]+ iters" | sed "s/^/pf=$pf /" | cut -c1-120
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_known_answers.py -q -x -k "gmres or arnoldi or graph" 2>&1 | tail -2
SFV_TIMING=1 timeout 900 python scripts/run_configs.py --cases c2 2>&1 | grep -E '"case"' | cut -c1-200
