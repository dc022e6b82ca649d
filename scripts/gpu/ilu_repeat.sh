# Soak of the streamed ILU sweep at C2 (scripts/probes/ilu_repeat.py): first and repeated applies
# after repeated setups against the sync-free sweep; variants (SFV_LIB) with injected delays
# (-DSFV_STREAM_DELAY=1/2/3, scripts/build_full_variant.py).
export PYTHONPATH=$PWD
export ILU_SEEDS=21,22
for v in ${VARIANTS:-default delay1 delay2 delay3}; do
  if [ $v = default ]; then unset SFV_LIB; else export SFV_LIB=scripts/probes/variants/libsfv_$v.so; fi
  echo "== $v"; timeout 900 python scripts/probes/ilu_repeat.py 2 20 2>&1 | tail -4 | cut -c1-160
done
