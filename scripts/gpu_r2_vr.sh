#!/bin/bash
# ViT 2D RoPE fused into the qkv GEMM epilogue: op test, engine parity, ViT pass fused vs separate kernel
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "rope" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_engine.py -q -x 2>&1 | tail -1
timeout 120 python __graft_entry__.py smoke 2>&1 | tail -1
for f in 1 0 1 0; do
  NOVA_VIT_ROPE_FUSED=$f python scripts/pass_profile.py --model 2b --stage vit --split 0 2>&1 | tail -1
done
NOVA_VIT_ROPE_FUSED=1 python scripts/pass_profile.py --model 2b --stage vit --split 24 2>&1 | tail -1
NOVA_VIT_ROPE_FUSED=0 python scripts/pass_profile.py --model 2b --stage vit --split 24 2>&1 | tail -1
