#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py -x -q 2>&1 | tail -3
timeout 300 python scripts/kbench.py --only gemv --iters 20 > gpurun_out/kb_gemv.jsonl 2>&1; grep -v '"B": 16' gpurun_out/kb_gemv.jsonl
timeout 100 python scripts/kbench.py --only attn
NOVA_PROFILER_RANGE=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --skip-profile --requests 4 --steps 1 --warmup 1 --no-compare > gpurun_out/bench_ncu.log 2>&1
tail -2 gpurun_out/bench_ncu.log | cut -c1-300; wc -l gpurun_out/launches.csv
