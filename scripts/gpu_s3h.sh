#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_engine.py -x -q 2>&1 | tail -2
timeout 1500 python bench.py --out gpurun_out/bench_s3h.json 2>gpurun_out/bench_s3h.err | tail -c 200; tail -3 gpurun_out/bench_s3h.err
