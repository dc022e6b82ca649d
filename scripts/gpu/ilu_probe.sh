timeout 300 python scripts/microbench.py --config c2 --what ilu --reps 10 2>&1 | tail -2
SFV_LIB=scripts/probes/variants/libsfv_probe32.so timeout 300 python scripts/microbench.py --config c2 --what ilu --reps 1 2>&1 | grep tri_stream | sort | uniq | head -8
