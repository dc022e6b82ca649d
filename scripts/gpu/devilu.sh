export PYTHONPATH=$PWD
SFV_TIMING=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -s -k "ilu" 2>&1 | grep -E "passed|failed|Error|error|assert|device ilu|c2 ilu1|declined" | head -30
SFV_TIMING=1 timeout 600 python scripts/run_configs.py --cases c2 2>&1 | grep -E '"case"|device ilu|declined' | cut -c1-400
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
