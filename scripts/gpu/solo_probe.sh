export PYTHONPATH=$PWD
SFV_LIB=scripts/probes/variants/libsfv_probe32.so timeout 300 python scripts/microbench.py --what ilu --reps 1 > gpurun_out/solo_probe.log 2>&1
grep "solo levels" gpurun_out/solo_probe.log | sort | uniq | awk '!seen[$2 $4 $6]++' | head -12
