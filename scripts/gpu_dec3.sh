#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "gemv_tma" 2>&1 | tail -2
timeout 600 python scripts/kbench.py --only gemv 2>/dev/null | grep gemv_tma | grep -v '"B": 16'
for S in 0 24 40 80; do timeout 120 python scripts/pass_profile.py --stage dec --B 2 --split $S 2>/dev/null; done
