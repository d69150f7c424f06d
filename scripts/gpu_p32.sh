#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_decode_fused.py tests/test_gpu_engine.py -x -q 2>&1 | tail -1
for m in 2b 7b; do for S in 0 40 80; do timeout 200 python scripts/pass_profile.py --model $m --stage dec --B 2 --split $S 2>/dev/null | sed "s/^{/{\"model\": \"$m\", /"; done; done
