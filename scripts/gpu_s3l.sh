#!/bin/bash
mkdir -p gpurun_out
T0=$(date +%s)
timeout 1500 python bench.py --out gpurun_out/bench_s3l.json 2>gpurun_out/bench_s3l.err | tail -c 200; echo; grep -i "stall\|error\|Traceback" gpurun_out/bench_s3l.err | head -3; tail -2 gpurun_out/bench_s3l.err
echo "bench wall $(( $(date +%s) - T0 )) s"
