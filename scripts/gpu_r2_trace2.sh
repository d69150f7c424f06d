#!/bin/bash
L=paper_2509_21301_b200
cp $L/libnova_trace.so $L/libnova.so
for m in 20 30; do
NOVA_UMMA_MASK=$m NOVA_UMMA_TRACE_N=17920 timeout 300 python scripts/umma_trace_pass.py --model 2b --s 24 32 64 0 2>&1 | grep span
done
NOVA_UMMA_MASK=30 NOVA_UMMA_TRACE_N=1536 timeout 300 python scripts/umma_trace_pass.py --model 2b --s 24 64 2>&1 | grep span
NOVA_UMMA_MASK=20 NOVA_UMMA_TRACE_N=151936 timeout 300 python scripts/umma_trace_pass.py --model 2b --s 24 2>&1 | grep span
cp $L/libnova_new.so $L/libnova.so
