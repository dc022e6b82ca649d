export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_gpu_adapter.py -q -s 2>&1 | tail -25
