#!/bin/bash
# One GPU round trip: parity tests, kernel micro-bench, default bench line.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -5 gpurun_out/pytest_gpu.log
timeout 600 python scripts/kbench.py --iters 20 > gpurun_out/kbench.jsonl 2> gpurun_out/kbench.err; tail -3 gpurun_out/kbench.err
timeout 1500 python bench.py --out gpurun_out/bench.json > gpurun_out/bench.log 2> gpurun_out/bench.err; tail -5 gpurun_out/bench.err
tail -c 600 gpurun_out/bench.log
