#!/bin/bash
mkdir -p gpurun_out
NCU="ncu --profile-from-start off --set full --clock-control none --import-source on"
for S in 0 32; do
timeout 600 $NCU -k regex:gemv_tma -c 2 -o gpurun_out/ncu_s3n_gemv2b_s$S -f python scripts/pass_profile.py --model 2b --stage dec --profile --split $S > /dev/null 2>&1
done
timeout 600 $NCU -k regex:decode_attn -c 1 -o gpurun_out/ncu_s3n_dattn2b -f python scripts/pass_profile.py --model 2b --stage dec --profile > /dev/null 2>&1
python scripts/ncu_summary.py gpurun_out/ncu_s3n_gemv2b_s0.ncu-rep gpurun_out/ncu_s3n_gemv2b_s32.ncu-rep gpurun_out/ncu_s3n_dattn2b.ncu-rep --out gpurun_out/r01_s3_ncu_full_dec2b.json
ls -la gpurun_out/*.ncu-rep
