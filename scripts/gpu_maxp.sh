#!/bin/bash
for M in 16 8 4 2; do echo "maxP $M"; NOVA_GEMV_MAXP=$M timeout 300 python scripts/dec_slice_probe.py --model 2b 2>&1 | grep "^{" | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d.get('s','full'), d.get('dec_solo_ms', d.get('full_ms')))" | tr '\n' ';'; echo; done
NOVA_GEMV_MAXP=4 timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum,launch__grid_size,dram__bytes_read.sum --clock-control none --csv --log-file gpurun_out/ll3_2b_s32_p4.csv python scripts/pass_profile.py --model 2b --stage dec --profile --split 32 > /dev/null 2>&1
for M in 16 4; do echo "7b maxP $M"; NOVA_GEMV_MAXP=$M timeout 300 python scripts/dec_slice_probe.py --model 7b 2>&1 | grep "^{" | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d.get('s','full'), d.get('dec_solo_ms', d.get('full_ms')))" | tr '\n' ';'; echo; done
