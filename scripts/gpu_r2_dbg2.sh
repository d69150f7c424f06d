#!/bin/bash
mkdir -p gpurun_out
for k in 2 4; do NOVA_DEC_FUSED_STOP=$k NOVA_DEC_FUSED_HALT=1 timeout 120 python tests/dbg_fused.py halt 2>&1 | grep -v Warn | tail -3; done
