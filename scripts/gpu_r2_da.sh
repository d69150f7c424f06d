#!/bin/bash
# decode attention ring depth by partition + per-kernel launch lists of 2B B=16 decode (full GPU / 24 SMs)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py -q -x 2>&1 | tail -2
for v in "NOVA_DA_NST=2" "NOVA_DA_NST=0"; do
  env $v NOVA_DEC_TMA=30 timeout 300 python scripts/dec_splits.py --model 2b --B 2 16 --splits 0 24 32 48 72 2>&1 | grep '^{'
  env $v NOVA_DEC_TMA=30 timeout 300 python scripts/dec_splits.py --model 7b --B 2 16 --splits 0 24 48 2>&1 | grep '^{'
done
for m in 30 31; do for S in 0 24; do
NOVA_DEC_TMA=30 NOVA_UMMA_MASK=$m timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum,launch__grid_size,dram__bytes_read.sum --clock-control none --csv --log-file gpurun_out/ll_2b_b16_m${m}_s$S.csv python scripts/pass_profile.py --model 2b --stage dec --profile --split $S --B 16 --iters 1 > /dev/null 2>&1
python scripts/ll_summary.py gpurun_out/ll_2b_b16_m${m}_s$S.csv | head -12
done; done
