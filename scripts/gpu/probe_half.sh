# Timing probes (wrong results): upper bounds of a face-once flux pass and of removing its arithmetic
export PYTHONPATH=$PWD
for lib in "" scripts/probes/variants/libsfv_half.so scripts/probes/variants/libsfv_nocomp.so scripts/probes/variants/libsfv_halfnc.so; do
  for r in 1 2; do
  SFV_LIB=$lib timeout 300 python scripts/microbench.py --config c2 --what jv --reps 400 2>&1 | grep -o '"jv_ms": [0-9.]*' | sed "s|^|${lib:-default} |"
  done
done
