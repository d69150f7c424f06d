#!/bin/bash
mkdir -p gpurun_out
/usr/bin/time -f "bench wall %e s" timeout 1500 python bench.py --out gpurun_out/bench_s3c.json 2>gpurun_out/bench_s3c.err | tail -c 300; tail -4 gpurun_out/bench_s3c.err
