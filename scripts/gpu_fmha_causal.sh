#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -k "flash_attn" 2>&1 | tail -5
timeout 200 python scripts/kbench.py --only attn 2>&1 | tee gpurun_out/kbench_attn_causal.jsonl
