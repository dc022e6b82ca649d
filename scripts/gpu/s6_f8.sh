# Session 6: the architecturally correct hand-over (release arrive, HBM stores behind it): timing and soak
export PYTHONPATH=$PWD
for v in "" f8 "" f8; do
  if [ -n "$v" ]; then export SFV_LIB=scripts/probes/variants/libsfv_$v.so; else unset SFV_LIB; fi
  echo "== variant ${v:-default}"
  timeout 300 python scripts/microbench.py --config c2 --what ilu --reps 20 2>&1 | grep -E "precond_apply" | sed 's/.*"precond_apply_ms_incl_sync"/apply_ms/' | head -3
done
unset SFV_LIB
REPS=1 ROUNDS=300 VARIANTS="d3f8 d7" bash scripts/gpu/s6_cold.sh
