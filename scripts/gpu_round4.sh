#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q 2>&1 | tail -3
timeout 300 python scripts/kbench.py --only gemv --iters 20 > gpurun_out/kb_gemv.jsonl 2>&1; cat gpurun_out/kb_gemv.jsonl
timeout 100 python scripts/kbench.py --only dattn
timeout 100 python scripts/kbench.py --only attn
timeout 300 python bench.py --skip-profile --requests 4 --steps 1 --warmup 1 --no-compare --out gpurun_out/bench_small.json 2>gpurun_out/bench_small.err; grep "launches before" gpurun_out/bench_small.err
N0=$(grep "launches before" gpurun_out/bench_small.err | grep -o "[0-9]*$")
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s $N0 -c 5000 --csv --log-file gpurun_out/launches.csv python bench.py --skip-profile --requests 4 --steps 1 --warmup 1 --no-compare > gpurun_out/bench_ncu.log 2>&1
tail -2 gpurun_out/bench_ncu.log; wc -l gpurun_out/launches.csv
