#!/bin/bash
# session-3 final validation: tests, smoke, 2B/7B solo passes, default bench (configs[1]), cfg3 bench, reference arm
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for M in 2b 7b; do for S in 0 32 64; do timeout 120 python scripts/pass_profile.py --model $M --stage dec --split $S 2>/dev/null; done; done > gpurun_out/pass_s3o.jsonl
timeout 300 python scripts/pass_profile.py --model 2b --stage vit,pre 2>/dev/null >> gpurun_out/pass_s3o.jsonl
cat gpurun_out/pass_s3o.jsonl
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum,launch__grid_size,dram__bytes_read.sum --clock-control none --csv --log-file gpurun_out/ll_s3o_2b_s0.csv python scripts/pass_profile.py --model 2b --stage dec --profile > /dev/null 2>&1
timeout 2400 python bench.py --out gpurun_out/bench_s3o.json 2>gpurun_out/bench_s3o.err | tail -c 200; echo; grep -i "stall\|error\|Traceback" gpurun_out/bench_s3o.err | head -3
timeout 2400 python bench.py --workload cfg3 --out gpurun_out/bench_s3o_cfg3.json 2>gpurun_out/bench_s3o_cfg3.err | tail -c 200; echo; grep -i "stall\|error\|Traceback" gpurun_out/bench_s3o_cfg3.err | head -3
