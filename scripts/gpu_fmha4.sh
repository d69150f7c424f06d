#!/bin/bash
mkdir -p gpurun_out
timeout 30 python scripts/attn_one.py 1286 28 4 128 1 && echo "causal ok"
timeout 30 python scripts/attn_one.py 4888 16 16 80 0 && echo "vit ok"
timeout 120 python -m pytest tests/test_gpu_kernels.py -x -q -k "flash_attn" 2>&1 | tail -2
for T in 1 0; do echo "v4 turn=$T"; NOVA_FMHA_TURN=$T timeout 60 python scripts/kbench.py --only attn 2>&1 | grep tc; done
timeout 120 ncu --set full --clock-control none --import-source on -k regex:fmha4 -s 3 -c 1 -o gpurun_out/ncu_fmha4b_vit python scripts/attn_one.py 4888 16 16 80 0 > /dev/null 2>&1
