export PYTHONPATH=$PWD
timeout 120 python /tmp/g.py 100 0 1 2>&1 | tail -2
