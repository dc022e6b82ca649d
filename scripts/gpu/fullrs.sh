export PYTHONPATH=$PWD
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -s -k "run_steps_matches_reference" 2>&1 | grep -E "newton|passed|failed|Error|assert" | head -20
