#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for S in 0 32 64; do timeout 120 python scripts/pass_profile.py --model 7b --stage dec --split $S 2>/dev/null; done
for B in 1 4 8 16; do timeout 120 python scripts/pass_profile.py --model 7b --stage dec --B $B 2>/dev/null; done
timeout 2400 python bench.py --workload cfg3 --out gpurun_out/bench_s3q_cfg3.json 2>gpurun_out/bench_s3q_cfg3.err | tail -c 200; echo; grep -i "stall\|error\|Traceback" gpurun_out/bench_s3q_cfg3.err | head -3
