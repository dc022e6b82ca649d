# Solo levels in the streamed ILU sweep: bitwise tests, then apply time with / without.
export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "ilu_apply_bitwise or sweep_modes or device_setup_bitwise or ilu_apply_transient or symmetry_patches or run_steps_parity" 2>&1 | tail -3
for v in default; do
  for hp in 0; do
    if [ $v = default ]; then unset SFV_LIB; else export SFV_LIB=scripts/probes/variants/libsfv_$v.so; fi
    if [ $hp = 1 ]; then export SFV_HOST_PRECOND=1; else unset SFV_HOST_PRECOND; fi
    timeout 300 python scripts/microbench.py --what ilu --reps 40 > gpurun_out/solo_${v}_$hp.log 2>gpurun_out/solo_${v}_$hp.err
    echo "$v host=$hp: $(grep -o '"precond_apply_ms_incl_sync": [0-9.]*' gpurun_out/solo_${v}_$hp.log) $(grep -o '"sweep": [0-9]*' gpurun_out/solo_${v}_$hp.log) $(tail -n 1 gpurun_out/solo_${v}_$hp.err | cut -c1-120)"
  done
done
