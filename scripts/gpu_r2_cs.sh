#!/bin/bash
# causal key split v2 (<= 4 chunks, merge with every chunk's 32-column slice in flight): tests + timings
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "flash" 2>&1 | tail -1
for c in 0 1; do
  echo "csplit=$c"; NOVA_FMHA_CSPLIT=$c timeout 300 python scripts/kbench.py --only attn --iters 20 2>&1 | grep -v mma | grep pre
  for m in 2b 7b; do NOVA_FMHA_CSPLIT=$c python scripts/pass_profile.py --model $m --stage pre --split 0 2>&1 | tail -1; done
done
timeout 900 python -m pytest tests/test_gpu_engine.py -q -x 2>&1 | tail -1
