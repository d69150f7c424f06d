#!/bin/bash
M=gpu__time_duration.sum,launch__grid_size
for u in 128 512; do
NOVA_UMMA_UNITS=$u timeout 600 ncu --profile-from-start off --metrics $M --csv --log-file gpurun_out/r2_ll_units$u.csv python scripts/pass_profile.py --model 2b --stage dec --profile > /dev/null 2>&1
done
python scripts/ll_summary.py gpurun_out/r2_ll_units128.csv gpurun_out/r2_ll_units512.csv
