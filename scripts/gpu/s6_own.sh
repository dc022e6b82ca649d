# Session 6: own [w | G] records of a tile staged with cp.async one tile ahead (flux pass)
export PYTHONPATH=$PWD
for v in ownoff "" ownoff ""; do
  if [ -n "$v" ]; then export SFV_LIB=scripts/probes/variants/libsfv_$v.so; else unset SFV_LIB; fi
  for c in c2 c4; do
  timeout 300 python scripts/microbench.py --config $c --what jv --reps 300 2>&1 | grep -o '"jv_ms": [0-9.]*' | sed "s/^/${v:-own} $c /"
  done
done
unset SFV_LIB
timeout 300 python scripts/jv_sweep.py --out gpurun_out/s6_jv_sweep.json 2>&1 | tail -3 | cut -c1-300
timeout 900 python -m pytest tests -m gpu -q -x -k "jv or residual or golden or fullsize or known or tet or host_buffers or transient" 2>&1 | tail -4
