#!/bin/bash
# causal FMHA key split: kernel times vs the split floor T (NOVA_FMHA_SPLIT: 0 = no split, 1 = auto, k = T >= k)
for sp in 0 1 10 16; do
  echo "split=$sp"; NOVA_FMHA_SPLIT=$sp timeout 300 python scripts/kbench.py --only attn --iters 20 2>&1 | grep -v mma | grep pre
done
