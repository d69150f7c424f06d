#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "flash" 2>&1 | tail -2
timeout 300 python scripts/kbench.py --only attn 2>&1 | grep vit | grep tc
NOVA_FMHA_SPLIT=0 timeout 300 python scripts/kbench.py --only attn 2>&1 | grep vit | grep tc
