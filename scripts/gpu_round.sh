#!/bin/bash
# One GPU call: kernel tests, kernel micro-benchmark, ncu launch list + full capture of top kernels.
set -x
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q 2>&1 | tail -3
timeout 300 python scripts/kbench.py --iters 20 > gpurun_out/kbench.jsonl 2>gpurun_out/kbench.err; tail -3 gpurun_out/kbench.err
cat gpurun_out/kbench.jsonl
# full ncu capture of one GEMV (gate_up, B=4) and one ViT GEMM and the ViT FMHA
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemv_kernel -s 40 -c 1 -o gpurun_out/ncu_gemv python scripts/kbench.py --only gemv --iters 3 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 6 -c 1 -o gpurun_out/ncu_gemm python scripts/kbench.py --only gemm --iters 3 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:flash_attn_kernel -s 3 -c 1 -o gpurun_out/ncu_fa python scripts/kbench.py --only attn --iters 3 > /dev/null 2>&1
ls -la gpurun_out
