# Session-6 probe of the ILU hand-over: one thread of CTA 5 stores to an untouched 2 MB page
# (a TLB miss in flight) just before (d4) / after (d5) its ring stores, every 8th level.
export PYTHONPATH=$PWD
export ILU_SEEDS=21
export SFV_ILU_WARMUP=0
for v in $VARIANTS; do
  if [ "$v" = base ]; then unset SFV_LIB; else export SFV_LIB=scripts/probes/variants/libsfv_$v.so; fi
  echo "== $v"; timeout 900 python scripts/probes/ilu_repeat.py ${REPS:-3} ${ROUNDS:-8} 2>&1 | tail -12 | cut -c1-160
done
