#!/bin/bash
# session-3 late: tests, smoke, 2B decode launch lists (full GPU and a 32-SM slice), default bench (configs[1])
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for S in 0 32; do
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum,launch__grid_size,dram__bytes_read.sum --clock-control none --csv --log-file gpurun_out/ll_s3l_2b_s$S.csv python scripts/pass_profile.py --model 2b --stage dec --profile --split $S > /dev/null 2>&1
done
for S in 0 32 64; do timeout 120 python scripts/pass_profile.py --model 2b --stage dec --split $S 2>/dev/null; done
timeout 2400 python bench.py --out gpurun_out/bench_s3l.json 2>gpurun_out/bench_s3l.err | tail -c 300; echo; grep -i "stall\|error\|Traceback" gpurun_out/bench_s3l.err | head -3
