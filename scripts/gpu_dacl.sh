#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_decode_fused.py -x -q -k "decode or attn" 2>&1 | tail -2
timeout 400 python scripts/dec_slice_probe.py --model 2b 2>&1 | grep "^{"
timeout 600 python -m pytest tests/test_gpu_engine.py -x -q 2>&1 | tail -2
timeout 120 python scripts/kbench.py --only dattn 2>&1 | tail -12
