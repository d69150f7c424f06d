#!/bin/bash
mkdir -p gpurun_out
for S in 32 0; do
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum,launch__grid_size,dram__bytes_read.sum --clock-control none --csv --log-file gpurun_out/ll_2b_s$S.csv python scripts/pass_profile.py --model 2b --stage dec --profile --split $S > /dev/null 2>&1
done
python scripts/pass_profile.py --model 2b --stage dec --split 32
python scripts/pass_profile.py --model 2b --stage dec --split 0
