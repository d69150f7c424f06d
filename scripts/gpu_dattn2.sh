#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_decode_fused.py -x -q -k "decode" 2>&1 | tail -1
timeout 100 python scripts/kbench.py --only dattn
for B in 2 8 16; do timeout 120 python scripts/pass_profile.py --stage dec --B $B 2>/dev/null; done
