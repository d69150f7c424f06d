#!/bin/bash
mkdir -p gpurun_out
NCU="ncu --profile-from-start off --set full --clock-control none --import-source on"
for S in 0 32; do
timeout 600 $NCU -k regex:decode_fused -c 1 -o gpurun_out/r2_ncu_fused_2b_s$S -f python scripts/pass_profile.py --model 2b --stage dec --profile --split $S > gpurun_out/r2_ncu_fused_2b_s$S.log 2>&1; echo "ncu s=$S rc=$?"
done
ls -la gpurun_out/*.ncu-rep
