#!/bin/bash
# CTA-pair GEMM: parity (all tile families) then per-tile throughput at the ViT / prefill shapes
mkdir -p gpurun_out
timeout 240 python -m pytest tests/test_gpu_kernels.py -x -q -k "gemm" 2>&1 | tail -5
timeout 300 python scripts/kbench.py --only gemm --gemm-modes 0,1,1256,1224,1192,1160,1128 > gpurun_out/kbench_gemm2.jsonl 2>&1; cat gpurun_out/kbench_gemm2.jsonl
