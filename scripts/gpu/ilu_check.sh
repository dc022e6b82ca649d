set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "ilu or precond or golden or stream or sweep" 2>&1 | tail -4
SFV_TIMING=1 timeout 600 python scripts/run_configs.py --cases c2 > gpurun_out/ilu_c2.log 2>&1
tail -3 gpurun_out/ilu_c2.log
