#!/bin/bash
# session-3 health check of HEAD: gpu tests, smoke, default bench, launch list
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -6
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1500 python bench.py --out gpurun_out/bench_s3a.json 2>gpurun_out/bench_s3a.err | tail -c 3000; tail -5 gpurun_out/bench_s3a.err
timeout 300 python scripts/kbench.py > gpurun_out/kbench_s3a.jsonl 2>&1; tail -30 gpurun_out/kbench_s3a.jsonl
