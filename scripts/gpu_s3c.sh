#!/bin/bash
mkdir -p gpurun_out
T0=$(date +%s)
timeout 1500 python bench.py --out gpurun_out/bench_s3c.json 2>gpurun_out/bench_s3c.err | tail -c 300; tail -4 gpurun_out/bench_s3c.err
echo "bench wall $(( $(date +%s) - T0 )) s"
