#!/bin/bash
mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none --import-source on -k regex:fmha3 -s 3 -c 1 -o gpurun_out/ncu_fmha_vit python scripts/attn_one.py 4888 16 16 80 0 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:fmha3 -s 3 -c 1 -o gpurun_out/ncu_fmha_pre python scripts/attn_one.py 1286 28 4 128 1 > /dev/null 2>&1
ls gpurun_out
