#!/bin/bash
L=paper_2509_21301_b200
cp $L/libnova_new.so $L/libnova.so
timeout 300 python -m pytest tests/test_gpu_gemv_umma.py -x -q 2>&1 | tail -3
for ck in 2 4; do
  echo "new ckmin=$ck"
  for sh in 2b_gu 2b_down 2b_o 2b_lm 7b_gu 7b_down; do NOVA_UMMA_CKMIN=$ck timeout 300 python scripts/ubench.py --only $sh --iters 20 2>&1 | grep '"B": 2'; done
  for m in 20 30; do NOVA_UMMA_CKMIN=$ck NOVA_UMMA_MASK=$m timeout 300 python scripts/dec_splits.py --model 2b --B 2 16 2>&1 | tail -2; done
  NOVA_UMMA_CKMIN=$ck NOVA_UMMA_MASK=30 timeout 300 python scripts/dec_splits.py --model 7b --B 2 2>&1 | tail -1
done
cp $L/libnova_old.so $L/libnova.so
echo old
for sh in 2b_gu 2b_down 2b_o 2b_lm 7b_gu 7b_down; do timeout 300 python scripts/ubench.py --only $sh --iters 20 2>&1 | grep '"B": 2'; done
NOVA_UMMA_MASK=20 timeout 300 python scripts/dec_splits.py --model 2b --B 2 16 2>&1 | tail -2
NOVA_UMMA_MASK=20 timeout 300 python scripts/dec_splits.py --model 7b --B 2 2>&1 | tail -1
cp $L/libnova_new.so $L/libnova.so
