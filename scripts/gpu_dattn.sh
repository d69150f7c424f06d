#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_decode_fused.py -x -q -k "decode" 2>&1 | tail -1
for S in 0 0 40 80; do timeout 120 python scripts/pass_profile.py --stage dec --B 2 --split $S 2>/dev/null; done
for B in 1 8; do timeout 120 python scripts/pass_profile.py --stage dec --B $B 2>/dev/null; done
