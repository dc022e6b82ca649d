export PYTHONPATH=$PWD
timeout 900 python -m pytest tests -m gpu -x -q -k "graph or host_buffers or run_steps or golden" 2>&1 | tail -4
SFV_TIMING=1 timeout 600 python scripts/run_configs.py --cases c1,c2 2>&1 | grep -o '"case": "c[12]".*"krylov_total": [0-9]*\|Error.*\|gmres graph.*'
