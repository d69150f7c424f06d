#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_decode_fused.py -x -q -k "gemv or decode" 2>&1 | tail -3
timeout 400 python scripts/dec_slice_probe.py --model 2b 2>&1 | grep "^{"
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum,launch__grid_size,dram__bytes_read.sum --clock-control none --csv --log-file gpurun_out/ll2_2b_s32.csv python scripts/pass_profile.py --model 2b --stage dec --profile --split 32 > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_engine.py -x -q 2>&1 | tail -3
