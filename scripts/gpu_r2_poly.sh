#!/bin/bash
# sweep EXP_POLY_OF_8 in the ViT/prefill FMHA (variant libraries built on the CPU host)
mkdir -p gpurun_out
L=paper_2509_21301_b200
for k in 2 1 3 4 5 2; do
  cp $L/libnova_p$k.so $L/libnova.so
  echo "poly=$k"
  timeout 60 python scripts/kbench.py --only attn 2>&1 | grep tc
  timeout 120 python -m pytest tests/test_gpu_kernels.py -x -q -k "flash_attn" 2>&1 | tail -1
done
