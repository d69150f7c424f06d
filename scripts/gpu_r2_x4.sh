#!/bin/bash
L=paper_2509_21301_b200
cp $L/libnova_new.so $L/libnova.so
timeout 300 python -m pytest tests/test_gpu_gemv_umma.py -x -q 2>&1 | tail -1
NOVA_UMMA_RING=1 timeout 300 python -m pytest tests/test_gpu_gemv_umma.py -x -q 2>&1 | tail -1
cp $L/libnova_trace.so $L/libnova.so
for r in 2 0; do NOVA_UMMA_RING=$r NOVA_UMMA_CKMIN=4 timeout 60 python scripts/umma_trace.py 17920 1536 3 24 2 2>&1 | tail -1; done
NOVA_UMMA_RING=0 NOVA_UMMA_CKMIN=4 NOVA_UMMA_MASK=30 NOVA_UMMA_TRACE_N=17920 timeout 300 python scripts/umma_trace_pass.py --model 2b --s 24 64 2>&1 | grep span
cp $L/libnova_new.so $L/libnova.so
for r in 0 1; do
  echo "ring=$r"
  for sh in 2b_gu 2b_lm 7b_gu 7b_down 2b_down 2b_o; do NOVA_UMMA_RING=$r NOVA_UMMA_CKMIN=4 timeout 300 python scripts/ubench.py --only $sh --iters 20 2>&1 | grep '"B": 2'; done
  for m in 20 30; do NOVA_UMMA_RING=$r NOVA_UMMA_CKMIN=4 NOVA_UMMA_MASK=$m timeout 300 python scripts/dec_splits.py --model 2b --B 2 16 2>&1 | tail -2; done
  NOVA_UMMA_RING=$r NOVA_UMMA_CKMIN=4 NOVA_UMMA_MASK=30 timeout 300 python scripts/dec_splits.py --model 7b --B 2 2>&1 | tail -1
done
