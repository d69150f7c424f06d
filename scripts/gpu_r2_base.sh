#!/bin/bash
# round 2 baseline: GPU tests + decode-on-a-slice probe (2B, 7B) on the round-1 code
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2_base_smi.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2_base_pytest.log 2>&1; tail -3 gpurun_out/r2_base_pytest.log
timeout 600 python scripts/dec_slice_probe.py --model 2b > gpurun_out/r2_base_slice2b.jsonl 2>gpurun_out/r2_base_slice2b.err
timeout 600 python scripts/dec_slice_probe.py --model 7b > gpurun_out/r2_base_slice7b.jsonl 2>gpurun_out/r2_base_slice7b.err
tail -2 gpurun_out/r2_base_slice2b.jsonl gpurun_out/r2_base_slice7b.jsonl
