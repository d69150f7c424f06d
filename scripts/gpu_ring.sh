#!/bin/bash
mkdir -p gpurun_out
NOVA_GEMV_RING=41 timeout 300 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_decode_fused.py -x -q -k "gemv or decode" 2>&1 | tail -2
for R in 22 41 31; do for S in 0 40 80; do
  NOVA_GEMV_RING=$R timeout 120 python scripts/pass_profile.py --stage dec --B 2 --split $S 2>/dev/null | sed "s/^{/{\"ring\": $R, /"
done; done
