export PYTHONPATH=$PWD
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -x -s -k "sequential or run_steps" 2>&1 | grep -v "^$" | tail -25
