#!/bin/bash
# configs[3]: layer-wise ViT offload (7B) on the session-3 code (fused-RoPE qkv GEMM on ring slots)
mkdir -p gpurun_out
timeout 1200 python scripts/offload_bench.py --model 7b --iters 5 > gpurun_out/r2_offload.json 2> gpurun_out/r2_offload.err; echo "rc=$?"
tail -c 2500 gpurun_out/r2_offload.json
tail -3 gpurun_out/r2_offload.err
