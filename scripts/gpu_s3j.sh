#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 100 python scripts/kbench.py --only attn 2>&1 | grep tc
for i in 1 2; do
timeout 1300 python bench.py --out gpurun_out/bench_s3j_$i.json 2>gpurun_out/bench_s3j_$i.err | tail -c 150; echo; grep -i "stall\|error\|Traceback" gpurun_out/bench_s3j_$i.err | head -3
done
