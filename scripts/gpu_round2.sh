#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py -x -q 2>&1 | tail -4
timeout 300 python scripts/kbench.py --iters 20 > gpurun_out/kbench2.jsonl 2>gpurun_out/kbench2.err; tail -3 gpurun_out/kbench2.err
cat gpurun_out/kbench2.jsonl
timeout 300 ncu --set full --clock-control none --import-source on -k regex:decode_attn_partial -s 2 -c 1 -o gpurun_out/ncu_dattn python scripts/kbench.py --only dattn --iters 3 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:fmha_tc -s 1 -c 1 -o gpurun_out/ncu_fmha python scripts/kbench.py --only attn --iters 2 > /dev/null 2>&1
timeout 600 python bench.py --requests 24 --steps 2 --warmup 1 --out gpurun_out/bench2.json 2>gpurun_out/bench2.err; tail -5 gpurun_out/bench2.err
