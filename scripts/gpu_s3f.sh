#!/bin/bash
# traffic per launch for the bench's kernel classes, then the full bench
mkdir -p gpurun_out
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
timeout 600 ncu --profile-from-start off --metrics $M --csv --log-file gpurun_out/traffic_dec.csv python scripts/pass_profile.py --stage dec --profile > /dev/null 2>&1
timeout 600 ncu --profile-from-start off --metrics $M --csv --log-file gpurun_out/traffic_vit.csv python scripts/pass_profile.py --stage vit --profile > /dev/null 2>&1
python scripts/ncu_traffic.py gpurun_out/traffic_dec.csv gpurun_out/traffic_vit.csv --out profiles/ncu_traffic.json
cp profiles/ncu_traffic.json gpurun_out/ncu_traffic.json
timeout 1500 python bench.py --out gpurun_out/bench_s3f.json 2>gpurun_out/bench_s3f.err | tail -c 200; tail -3 gpurun_out/bench_s3f.err
