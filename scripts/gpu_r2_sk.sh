#!/bin/bash
# stream-K gemv_umma: parity, micro-bench and decode iterations on partitions vs the previous kernel
mkdir -p gpurun_out
L=paper_2509_21301_b200
cp $L/libnova_new.so $L/libnova.so
timeout 300 python -m pytest tests/test_gpu_gemv_umma.py -x -q 2>&1 | tail -3
for v in old new; do
  cp $L/libnova_$v.so $L/libnova.so
  echo "== $v"
  timeout 300 python scripts/ubench.py --only 2b --iters 20 2>&1 | grep '"B": 2'
  timeout 200 python scripts/ubench.py --only 7b --iters 20 2>&1 | grep '"B": 2'
  for m in 20 30; do
    NOVA_UMMA_MASK=$m timeout 300 python scripts/dec_splits.py --model 2b --B 2 16 2>&1 | tail -2
  done
  NOVA_UMMA_MASK=20 timeout 300 python scripts/dec_splits.py --model 7b --B 2 2>&1 | tail -1
  NOVA_UMMA_MASK=30 timeout 300 python scripts/dec_splits.py --model 7b --B 2 2>&1 | tail -1
done
cp $L/libnova_new.so $L/libnova.so
