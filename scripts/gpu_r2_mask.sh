#!/bin/bash
L=paper_2509_21301_b200
cp $L/libnova_new.so $L/libnova.so
for m in 20 22 28 30; do
  NOVA_UMMA_CKMIN=4 NOVA_UMMA_MASK=$m timeout 300 python scripts/dec_splits.py --model 2b --B 2 8 16 --splits 0 24 32 40 48 56 64 72 2>&1 | tail -3
  NOVA_UMMA_CKMIN=4 NOVA_UMMA_MASK=$m timeout 300 python scripts/dec_splits.py --model 7b --B 2 16 --splits 0 24 32 48 64 72 2>&1 | tail -2
done
for ck in 2 8; do
  NOVA_UMMA_CKMIN=$ck NOVA_UMMA_MASK=30 timeout 300 python scripts/dec_splits.py --model 2b --B 2 16 --splits 0 24 32 40 48 56 64 72 2>&1 | tail -2
done
cp $L/libnova_old.so $L/libnova.so
NOVA_UMMA_MASK=20 timeout 300 python scripts/dec_splits.py --model 2b --B 2 8 16 --splits 0 24 32 40 48 56 64 72 2>&1 | tail -3
NOVA_UMMA_MASK=20 timeout 300 python scripts/dec_splits.py --model 7b --B 2 16 --splits 0 24 32 48 64 72 2>&1 | tail -2
cp $L/libnova_new.so $L/libnova.so
