#!/bin/bash
for S in 0 24; do
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launch_dec_s$S.csv python scripts/pass_profile.py --stage dec --split $S --profile > /dev/null 2>&1
python scripts/ncu_summary.py --launches gpurun_out/launch_dec_s$S.csv --out gpurun_out/launch_dec_s$S.json > /dev/null
python -c "
import json; d=json.load(open('gpurun_out/launch_dec_s$S.json'))['launches']
print('split $S total', sum(x['total_us'] for x in d)/2)
for x in d: print(x)"
done
