#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "flash or rope or norm" 2>&1 | tail -5
timeout 300 python scripts/kbench.py --only attn
timeout 300 python scripts/pass_profile.py --stage vit,pre 2>/dev/null
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launch_vit.csv python scripts/pass_profile.py --stage vit --profile > /dev/null 2>&1
python scripts/ncu_summary.py --launches gpurun_out/launch_vit.csv --out gpurun_out/launch_vit.json > /dev/null
python -c "
import json; d=json.load(open('gpurun_out/launch_vit.json'))['launches']
for x in d: print(x)"
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:fmha3 -c 1 -o gpurun_out/ncu_vit_fmha3 -f python scripts/pass_profile.py --stage vit --profile > /dev/null 2>&1
ls gpurun_out
