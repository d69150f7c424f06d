#!/bin/bash
# prefill RMSNorm fold (R25 on the GEMMs): kernel + engine parity, prefill pass times (fold on / off)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py -q -x 2>&1 | tail -3
timeout 120 python __graft_entry__.py smoke 2>&1 | tail -1
for f in 1 0; do for m in 2b 7b; do
  NOVA_FOLD_NORM=$f python scripts/pass_profile.py --model $m --stage pre --split 0 2>&1 | tail -1
done; done
