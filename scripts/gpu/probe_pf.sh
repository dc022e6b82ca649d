# flux pass with L2 prefetch of the next tile's records (SFV_FLUX_PF variants)
export PYTHONPATH=$PWD
for c in c2 c4; do
for lib in "" scripts/probes/variants/libsfv_pf1.so scripts/probes/variants/libsfv_pf2.so; do
  for r in 1 2; do
  SFV_LIB=$lib timeout 300 python scripts/microbench.py --config $c --what jv --reps 400 2>&1 | grep -o '"jv_ms": [0-9.]*' | sed "s|^|$c ${lib:-default} |"
  done
done
done
