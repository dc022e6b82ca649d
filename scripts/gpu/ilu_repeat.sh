# Soak of the streamed ILU sweep at C2 (scripts/probes/ilu_repeat.py): first applies after repeated
# setups against the sync-free sweep; optional variants (SFV_LIB) with injected delays.
export PYTHONPATH=$PWD
export ILU_SEEDS=21,22
for v in default delay1 delay2; do
  if [ $v = default ]; then unset SFV_LIB; else export SFV_LIB=scripts/probes/variants/libsfv_$v.so; fi
  echo "== $v"; timeout 900 python scripts/probes/ilu_repeat.py 2 20 2>&1 | tail -4 | cut -c1-160
done
