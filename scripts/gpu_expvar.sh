#!/bin/bash
# FMHA exp split sweep: libs built with EXP_POLY_OF_8 = 1..4 (build/var/)
mkdir -p gpurun_out
for R in 1 2; do for P in 1 2 3 4; do
  cp build/var/libnova_p$P.so paper_2509_21301_b200/libnova.so
  echo "poly=$P rep=$R"; timeout 90 python scripts/kbench.py --only attn 2>&1 | grep flash_attn_tc
done; done
cp build/var/libnova_p2.so paper_2509_21301_b200/libnova.so
