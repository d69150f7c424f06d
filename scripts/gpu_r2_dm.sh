#!/bin/bash
# decode attention: cluster merge spread over the ranks; partition-share stats test
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "decode" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_engine.py -q -x -k "partition_share or coexec or tiny" 2>&1 | tail -1
timeout 300 python scripts/dec_splits.py --model 2b --B 2 8 16 --splits 0 24 48 72 2>&1 | grep '^{'
timeout 300 python scripts/dec_splits.py --model 7b --B 2 16 --splits 0 24 48 2>&1 | grep '^{'
