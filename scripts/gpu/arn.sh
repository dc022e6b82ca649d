export PYTHONPATH=$PWD
SFV_GMRES_GRAPH=0 SFV_TIMING=1 timeout 300 python scripts/microbench.py --config c2 --what gmres --reps 1 2>&1 | grep -E "gmres [0-9]+ iters|device ilu|ms_per_iter" | cut -c1-200
SFV_GMRES_GRAPH=0 SFV_TIMING=1 timeout 300 python scripts/microbench.py --config c2 --what gmres --reps 1 2>&1 | grep -E "gmres [0-9]+ iters" | cut -c1-200
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_known_answers.py -q -x -k "gmres or arnoldi or graph" 2>&1 | tail -2
SFV_TIMING=1 timeout 900 python scripts/run_configs.py --cases c2 2>&1 | grep -E '"case"|device ilu' | cut -c1-220
