#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "flash" 2>&1 | tail -3
timeout 300 python scripts/kbench.py --only attn
timeout 300 python scripts/pass_profile.py --stage vit 2>/dev/null
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:fmha3 -c 1 -o gpurun_out/ncu_vit_fmha3 -f python scripts/pass_profile.py --stage vit --profile > /dev/null 2>&1
