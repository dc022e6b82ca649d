# Coupled (oblique symmetry plane) preconditioner tests.
export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "oblique" 2>&1 | tail -40
