#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_decode_fused.py -x -q -k "decode" 2>&1 | tail -2
timeout 100 python scripts/kbench.py --only dattn
for S in 0 40 80; do timeout 120 python scripts/pass_profile.py --stage dec --B 2 --split $S 2>/dev/null; done
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launch_dec40.csv python scripts/pass_profile.py --stage dec --split 40 --profile > /dev/null 2>&1
python scripts/ncu_summary.py --launches gpurun_out/launch_dec40.csv --out gpurun_out/launch_dec40.json > /dev/null
python -c "
import json; d=json.load(open('gpurun_out/launch_dec40.json'))['launches']
print('total', sum(x['total_us'] for x in d))
for x in d: print(x)"
