#!/bin/bash
# gemv_umma whole-block threshold (grid only, never the sums): default 128 vs stream-K everywhere
for w in 128 100000; do
  NOVA_UMMA_WBMIN=$w timeout 300 python scripts/dec_splits.py --model 2b --B 2 16 --splits 0 72 96 2>&1 | grep '^{'
  NOVA_UMMA_WBMIN=$w timeout 300 python scripts/dec_splits.py --model 7b --B 2 16 --splits 0 72 2>&1 | grep '^{'
done
