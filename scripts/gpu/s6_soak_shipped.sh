# Session 6: soak of the shipped sweep (no perturbation): first applies after a setup against the
# sync-free sweep, with the setup's warm-up apply (as shipped) and without it.
export PYTHONPATH=$PWD
export ILU_SEEDS=21
unset SFV_LIB
echo "== shipped (warm-up on)"; timeout 1500 python scripts/probes/ilu_repeat.py 1 ${ROUNDS_ON:-1500} 2>&1 | tail -4 | cut -c1-160
export SFV_ILU_WARMUP=0
echo "== warm-up off"; timeout 1500 python scripts/probes/ilu_repeat.py 1 ${ROUNDS_OFF:-3000} 2>&1 | tail -4 | cut -c1-160
