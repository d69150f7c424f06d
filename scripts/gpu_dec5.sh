#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
for S in 0 24 40 80; do timeout 120 python scripts/pass_profile.py --stage dec --B 2 --split $S 2>/dev/null; done | tee gpurun_out/pass_dec.jsonl
for B in 1 4 8 16; do timeout 120 python scripts/pass_profile.py --stage dec --B $B 2>/dev/null; done | tee -a gpurun_out/pass_dec.jsonl
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launch_dec.csv python scripts/pass_profile.py --stage dec --profile > /dev/null 2>&1
python scripts/ncu_summary.py --launches gpurun_out/launch_dec.csv --out gpurun_out/launch_dec.json > /dev/null
python -c "
import json; d=json.load(open('gpurun_out/launch_dec.json'))['launches']
print('total', sum(x['total_us'] for x in d)/2)
for x in d: print(x)"
