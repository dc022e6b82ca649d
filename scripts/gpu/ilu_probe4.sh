export PYTHONPATH=$PWD
for v in p16 p20 p4; do
  export SFV_LIB=scripts/probes/variants/libsfv_$v.so
  timeout 300 python scripts/microbench.py --config c2 --what ilu --reps 60 2>&1 | grep -o '"precond_apply_ms_incl_sync": [0-9.]*' | sed "s/^/$v /"
done
export SFV_LIB=scripts/probes/variants/libsfv_p32.so
timeout 300 python scripts/microbench.py --config c2 --what ilu --reps 2 2>&1 | grep "tri_stream" | sort | uniq -c | head -8
