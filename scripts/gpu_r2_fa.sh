#!/bin/bash
# causal FMHA key split (prefill) + vectorized RoPE/KV kernel: tests, prefill pass times, launch list
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py tests/test_gpu_chunk_attn.py -q -x 2>&1 | tail -2
for m in 2b 7b; do
  python scripts/pass_profile.py --model $m --stage pre --split 0 2>&1 | tail -1
done
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum,launch__grid_size,dram__bytes_read.sum --clock-control none --csv --log-file gpurun_out/ll_2b_pre2.csv python scripts/pass_profile.py --model 2b --stage pre --profile --split 0 --iters 1 > /dev/null 2>&1
python scripts/ll_summary.py gpurun_out/ll_2b_pre2.csv | head -12
