#!/bin/bash
# ncu --set full of the decode gate|up GEMV (gemv_umma EPI_BF16_SILUMUL, the largest decode linear) on the
# whole GPU and on a 24-SM green-context slice (2B, B = 2): the dominant class's biggest member
mkdir -p gpurun_out
NCU="ncu --profile-from-start off --set full --clock-control none --import-source on"
for S in 0 24; do
  timeout 600 $NCU -k regex:gemv_umma -s 2 -c 1 -o gpurun_out/rf_ncu_gu_2b_s$S -f python scripts/pass_profile.py --model 2b --stage dec --profile --split $S > /dev/null 2>&1
  echo "s=$S rc=$?"
done
python scripts/ncu_summary.py gpurun_out/rf_ncu_gu_2b_s0.ncu-rep gpurun_out/rf_ncu_gu_2b_s24.ncu-rep --out gpurun_out/rf_ncu_full_gu.json
cat gpurun_out/rf_ncu_full_gu.json | head -40
