export PYTHONPATH=$PWD
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -q -s -k "run_steps_matches_reference and c3" 2>&1 | grep -v "^$" | tail -8
