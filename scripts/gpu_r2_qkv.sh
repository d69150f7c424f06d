#!/bin/bash
# R25 ln1 fold + decode qkv on gemv_umma: op/engine parity, then decode iteration times per variant.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemv_umma.py tests/test_gpu_engine.py tests/test_gpu_decode_fused.py -q -x > gpurun_out/qkv_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/qkv_pytest.log
timeout 120 python __graft_entry__.py smoke 2>&1 | tail -1
for v in "NOVA_UMMA_MASK=30" "NOVA_UMMA_MASK=31" "NOVA_UMMA_MASK=31 NOVA_DEC_TMA=30"; do
  env $v timeout 300 python scripts/dec_splits.py --model 2b --B 2 16 --splits 0 24 32 48 72 2>&1 | grep '^{'
done
for v in "NOVA_UMMA_MASK=30" "NOVA_UMMA_MASK=31"; do
  env $v timeout 300 python scripts/dec_splits.py --model 7b --B 2 16 --splits 0 24 32 48 72 2>&1 | grep '^{'
done
