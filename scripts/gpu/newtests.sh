export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "symmetry_patches_host or odd_n" 2>&1 | tail -3
