#!/bin/bash
L=paper_2509_21301_b200
cp $L/libnova_trace.so $L/libnova.so
for r in 2 0; do for d in 0 1 2; do
  NOVA_UMMA_RING=$r NOVA_UMMA_DBG=$d NOVA_UMMA_CKMIN=4 timeout 60 python scripts/umma_trace.py 17920 1536 3 24 2 2>&1 | tail -1
done; done
for d in 0 1; do NOVA_UMMA_RING=0 NOVA_UMMA_DBG=$d NOVA_UMMA_CKMIN=4 NOVA_UMMA_MASK=30 NOVA_UMMA_TRACE_N=17920 timeout 300 python scripts/umma_trace_pass.py --model 2b --s 24 2>&1 | grep span; done
cp $L/libnova_new.so $L/libnova.so
