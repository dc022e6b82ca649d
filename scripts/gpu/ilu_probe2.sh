export PYTHONPATH=$PWD
for v in "" nostore nofence nofencestore ""; do
  if [ -n "$v" ]; then export SFV_LIB=scripts/probes/variants/libsfv_$v.so; else unset SFV_LIB; fi
  timeout 300 python scripts/microbench.py --config c2 --what ilu --reps 60 2>&1 | grep -o '"precond_apply_ms_incl_sync": [0-9.]*' | sed "s/^/${v:-default} /"
done
