export PYTHONPATH=$PWD
SFV_HEAVY=1 timeout 2400 python -m pytest tests/test_gpu_fullsize.py -q -s -k "full_solve_bit_identical" 2>&1 | grep -v "^$" | tail -25 | tee gpurun_out/seq_heavy.log
