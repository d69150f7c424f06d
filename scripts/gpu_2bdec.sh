#!/bin/bash
mkdir -p gpurun_out
timeout 300 python scripts/pass_profile.py --model 2b --stage dec --B 2 2>/dev/null
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launch_2bdec.csv python scripts/pass_profile.py --model 2b --stage dec --profile > /dev/null 2>&1
python scripts/ncu_summary.py --launches gpurun_out/launch_2bdec.csv --out gpurun_out/launch_2bdec.json > /dev/null
python -c "
import json; d=json.load(open('gpurun_out/launch_2bdec.json'))['launches']
print('total', sum(x['total_us'] for x in d))
for x in d: print(x)"
