export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_gpu_known_answers.py -q -x 2>&1 | tail -25
