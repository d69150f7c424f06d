#!/bin/bash
# norm-stat loads batched (gemv_umma); decode splits; 2B prefill + ViT launch lists (solo, full GPU)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_gemv_umma.py -q -x 2>&1 | tail -1
NOVA_DEC_TMA=30 timeout 300 python scripts/dec_splits.py --model 2b --B 2 16 --splits 0 24 32 48 72 2>&1 | grep '^{'
NOVA_DEC_TMA=30 timeout 300 python scripts/dec_splits.py --model 7b --B 2 16 --splits 0 24 48 72 2>&1 | grep '^{'
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum,launch__grid_size,dram__bytes_read.sum --clock-control none --csv --log-file gpurun_out/ll_2b_pre.csv python scripts/pass_profile.py --model 2b --stage pre --profile --split 0 --iters 1 > /dev/null 2>&1
python scripts/ll_summary.py gpurun_out/ll_2b_pre.csv | head -16
python scripts/pass_profile.py --model 2b --stage pre --split 0 2>&1 | tail -3
