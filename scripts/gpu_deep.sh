#!/bin/bash
mkdir -p gpurun_out
NOVA_GEMV_WIDE=1 timeout 300 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_decode_fused.py -x -q -k "gemv or decode" 2>&1 | tail -1
for D in 0 1; do for S in 0 40 80; do
  NOVA_GEMV_WIDE=$D timeout 120 python scripts/pass_profile.py --stage dec --B 2 --split $S 2>/dev/null | sed "s/^{/{\"deep\": $D, /"
done; done
NOVA_GEMV_WIDE=1 timeout 120 python scripts/pass_profile.py --stage dec --B 8 2>/dev/null
NOVA_GEMV_WIDE=1 timeout 120 python scripts/pass_profile.py --stage dec --B 16 2>/dev/null
