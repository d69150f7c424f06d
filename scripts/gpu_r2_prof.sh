#!/bin/bash
# round 2 profiling: per-class DRAM traffic (2B, 7B decode + ViT), decode launch lists (full GPU / 32-SM
# slice), ncu full captures of the tcgen05 decode GEMV (2B gate|up) on the full GPU and a 32-SM slice
mkdir -p gpurun_out
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,launch__grid_size
cp profiles/ncu_traffic.json gpurun_out/ncu_traffic.json
for mdl in 2b 7b; do
  timeout 600 ncu --profile-from-start off --metrics $M --csv --log-file gpurun_out/r2_traffic_${mdl}_dec.csv python scripts/pass_profile.py --model $mdl --stage dec --profile > /dev/null 2>&1
  timeout 600 ncu --profile-from-start off --metrics $M --csv --log-file gpurun_out/r2_traffic_${mdl}_vit.csv python scripts/pass_profile.py --model $mdl --stage vit --profile > /dev/null 2>&1
  python scripts/ncu_traffic.py gpurun_out/r2_traffic_${mdl}_dec.csv gpurun_out/r2_traffic_${mdl}_vit.csv --out gpurun_out/ncu_traffic.json --model qwen2vl-$mdl
done
timeout 600 ncu --profile-from-start off --metrics $M --csv --log-file gpurun_out/r2_ll_2b_dec_s32.csv python scripts/pass_profile.py --model 2b --stage dec --profile --split 32 > /dev/null 2>&1
python scripts/ll_summary.py gpurun_out/r2_traffic_2b_dec.csv gpurun_out/r2_ll_2b_dec_s32.csv gpurun_out/r2_traffic_7b_dec.csv > gpurun_out/r2_launch_dec_summary.txt 2>&1
NCU="ncu --profile-from-start off --set full --clock-control none --import-source on"
for S in 0 32; do
  timeout 600 $NCU -k regex:gemv_umma -c 1 -o gpurun_out/r2_ncu_umma_2b_s$S -f python scripts/pass_profile.py --model 2b --stage dec --profile --split $S > /dev/null 2>&1
done
python scripts/ncu_summary.py gpurun_out/r2_ncu_umma_2b_s0.ncu-rep gpurun_out/r2_ncu_umma_2b_s32.ncu-rep --out gpurun_out/r2_ncu_full_umma.json
ls gpurun_out/ | grep r2_
cat gpurun_out/r2_launch_dec_summary.txt | head -40
