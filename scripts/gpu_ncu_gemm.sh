#!/bin/bash
mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 3 -c 1 -o gpurun_out/ncu_gemm_fc1_pair python scripts/gemm_one.py 4888 5120 1280 1 1256 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 3 -c 1 -o gpurun_out/ncu_gemm_fc1_cta1 python scripts/gemm_one.py 4888 5120 1280 1 256 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 3 -c 1 -o gpurun_out/ncu_gemm_down_pair python scripts/gemm_one.py 1286 3584 18944 4 0 > /dev/null 2>&1
ls -la gpurun_out
