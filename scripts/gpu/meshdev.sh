export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -s -k "device_tet_mesh" 2>&1 | grep -E "passed|failed|Error|assert|c5 n=160|differ" | head -20
