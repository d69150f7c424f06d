#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_gemv_umma.py -x -q 2>&1 | tail -2
timeout 900 python scripts/ubench.py --only 2b 2>&1 | grep "^{"
for u in 1; do
NOVA_DEC_UMMA=$u timeout 300 python scripts/dec_slice_probe.py --model 2b 2>&1 | grep "^{" | tr '\n' ' '; echo " <- umma=$u"
done
