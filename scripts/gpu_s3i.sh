#!/bin/bash
mkdir -p gpurun_out
timeout 200 python -m pytest tests/test_gpu_kernels.py -x -q -k "flash_attn" 2>&1 | tail -1
timeout 100 python scripts/kbench.py --only attn 2>&1 | grep tc
timeout 1300 python bench.py --out gpurun_out/bench_s3i.json 2>gpurun_out/bench_s3i.err | tail -c 300; grep -v "^\[bench\]" gpurun_out/bench_s3i.err | tail -5; tail -2 gpurun_out/bench_s3i.err
