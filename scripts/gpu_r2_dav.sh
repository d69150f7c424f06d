#!/bin/bash
# virtual-CTA decode attention (fewer physical CTAs per (request, KV head) on small partitions) + RoPE/KV kernel
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py tests/test_gpu_chunk_attn.py -q -x 2>&1 | tail -2
for v in 0 1 2; do
  NOVA_DA_V=$v timeout 300 python scripts/dec_splits.py --model 2b --B 2 8 16 --splits 0 16 24 32 48 72 2>&1 | grep '^{'
  NOVA_DA_V=$v timeout 300 python scripts/dec_splits.py --model 7b --B 8 16 --splits 0 16 24 48 2>&1 | grep '^{'
done
python scripts/pass_profile.py --model 2b --stage pre --split 0 2>&1 | tail -1
