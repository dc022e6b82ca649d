export PYTHONPATH=$PWD
for i in 1 2 3; do timeout 300 python scripts/run_configs.py --cases c1,c2 2>&1 | grep -o '"case": "c[12]".*"newton": \[[0-9]*\]\|Error.*' | cut -c1-200; done
for i in 1 2; do SFV_GMRES_GRAPH=0 timeout 300 python scripts/run_configs.py --cases c1,c2 2>&1 | grep -o '"case": "c[12]".*"newton": \[[0-9]*\]\|Error.*' | cut -c1-200; done
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -5
