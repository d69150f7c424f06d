#!/bin/bash
mkdir -p gpurun_out
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
timeout 600 ncu --profile-from-start off --metrics $M --csv --log-file gpurun_out/traffic2b_dec.csv python scripts/pass_profile.py --model 2b --stage dec --profile > /dev/null 2>&1
timeout 600 ncu --profile-from-start off --metrics $M --csv --log-file gpurun_out/traffic2b_vit.csv python scripts/pass_profile.py --model 2b --stage vit --profile > /dev/null 2>&1
cp profiles/ncu_traffic.json gpurun_out/ncu_traffic.json
python scripts/ncu_traffic.py gpurun_out/traffic2b_dec.csv gpurun_out/traffic2b_vit.csv --out gpurun_out/ncu_traffic.json --model qwen2vl-2b
