export PYTHONPATH=$PWD
export ILU_SEEDS=21
for v in $VARIANTS; do
  export SFV_LIB=scripts/probes/variants/libsfv_$v.so
  echo "== $v"; timeout 900 python scripts/probes/ilu_repeat.py 1 40 2>&1 | tail -3 | cut -c1-140
done
