#!/bin/bash
# column-major split partials (coalesced): FMHA tests; ViT + causal kernel times; prefill with / without the causal split
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "flash" 2>&1 | tail -1
NOVA_FMHA_CSPLIT=1 timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "flash" 2>&1 | tail -1
for c in 0 1; do
  echo "csplit=$c"; NOVA_FMHA_CSPLIT=$c timeout 300 python scripts/kbench.py --only attn --iters 20 2>&1 | grep -v mma
  for m in 2b 7b; do NOVA_FMHA_CSPLIT=$c python scripts/pass_profile.py --model $m --stage pre --split 0 2>&1 | tail -1; done
done
python scripts/pass_profile.py --model 2b --stage vit --split 0 2>&1 | tail -1
