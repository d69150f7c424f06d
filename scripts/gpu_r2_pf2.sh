#!/bin/bash
# prefill fold with the row scale hoisted before the accumulator wait; then the L2 evict-first experiment
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "fold or gemm" 2>&1 | tail -1
for f in 1 0; do for m in 2b 7b; do
  NOVA_FOLD_NORM=$f python scripts/pass_profile.py --model $m --stage pre --split 0 2>&1 | tail -1
done; done
bash scripts/gpu_r2_ef.sh
