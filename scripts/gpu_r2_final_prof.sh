#!/bin/bash
# Round-2 final profiles on the final code: per-class DRAM traffic (2B / 7B decode + ViT) -> ncu_traffic.json
# (the bench's roofline `traffic`), decode launch lists (2B full GPU / 24-SM slice, 7B full GPU), the bench
# command's launch list (ncu, profiler range = the timed region), ncu --set full of the decode GEMV.
mkdir -p gpurun_out
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,launch__grid_size
cp profiles/ncu_traffic.json gpurun_out/ncu_traffic.json
for mdl in 2b 7b; do
  timeout 600 ncu --profile-from-start off --metrics $M --csv --log-file gpurun_out/rf_traffic_${mdl}_dec.csv python scripts/pass_profile.py --model $mdl --stage dec --profile > /dev/null 2>&1
  timeout 600 ncu --profile-from-start off --metrics $M --csv --log-file gpurun_out/rf_traffic_${mdl}_vit.csv python scripts/pass_profile.py --model $mdl --stage vit --profile > /dev/null 2>&1
  python scripts/ncu_traffic.py gpurun_out/rf_traffic_${mdl}_dec.csv gpurun_out/rf_traffic_${mdl}_vit.csv --out gpurun_out/ncu_traffic.json --model qwen2vl-$mdl
done
timeout 600 ncu --profile-from-start off --metrics $M --csv --log-file gpurun_out/rf_ll_2b_dec_s24.csv python scripts/pass_profile.py --model 2b --stage dec --profile --split 24 > /dev/null 2>&1
timeout 600 ncu --profile-from-start off --metrics $M --csv --log-file gpurun_out/rf_ll_2b_pre.csv python scripts/pass_profile.py --model 2b --stage pre --profile --iters 1 > /dev/null 2>&1
python scripts/ll_summary.py gpurun_out/rf_traffic_2b_dec.csv gpurun_out/rf_ll_2b_dec_s24.csv gpurun_out/rf_traffic_7b_dec.csv gpurun_out/rf_ll_2b_pre.csv gpurun_out/rf_traffic_2b_vit.csv > gpurun_out/rf_launch_summary.txt 2>&1
NOVA_PROFILER_RANGE=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/rf_launches_bench.csv python bench.py --skip-profile --requests 4 --steps 1 --warmup 1 --no-compare --no-solo-7b > gpurun_out/rf_bench_ncu.log 2>&1
python scripts/ncu_summary.py --launches gpurun_out/rf_launches_bench.csv --out gpurun_out/rf_launches_bench.json > /dev/null 2>&1
NCU="ncu --profile-from-start off --set full --clock-control none --import-source on"
for S in 0 24; do
  timeout 600 $NCU -k regex:gemv_umma -c 1 -o gpurun_out/rf_ncu_umma_2b_s$S -f python scripts/pass_profile.py --model 2b --stage dec --profile --split $S > /dev/null 2>&1
done
python scripts/ncu_summary.py gpurun_out/rf_ncu_umma_2b_s0.ncu-rep gpurun_out/rf_ncu_umma_2b_s24.ncu-rep --out gpurun_out/rf_ncu_full_umma.json
ls gpurun_out/ | grep rf_
head -60 gpurun_out/rf_launch_summary.txt
