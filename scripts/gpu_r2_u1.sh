#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_gemv_umma.py -x -q 2>&1 | tail -15
for u in 0 1; do
NOVA_DEC_UMMA=$u timeout 300 python scripts/dec_slice_probe.py --model 2b 2>&1 | grep "^{" | head -8 | tr '\n' ' '; echo " <- umma=$u"
done
