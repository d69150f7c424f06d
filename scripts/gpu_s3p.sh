#!/bin/bash
mkdir -p gpurun_out
NCU="ncu --profile-from-start off --set full --clock-control none --import-source on"
for S in 0 32; do
timeout 600 $NCU -k regex:gemv_tma -c 2 -o gpurun_out/ncu_s3p_gemv2b_s$S -f python scripts/pass_profile.py --model 2b --stage dec --profile --split $S > /dev/null 2>&1
done
python scripts/ncu_summary.py gpurun_out/ncu_s3p_gemv2b_s0.ncu-rep gpurun_out/ncu_s3p_gemv2b_s32.ncu-rep gpurun_out/ncu_s3n_dattn2b.ncu-rep --out gpurun_out/r01_s3_ncu_full_dec2b.json > /dev/null 2>&1
for MM in "2b 28" "2b 30" "2b 31" "7b 28" "7b 30" "7b 31"; do set -- $MM; echo "$1 mask $2"; NOVA_DEC_TMA=$2 timeout 300 python scripts/dec_slice_probe.py --model $1 2>&1 | grep "^{" | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d.get('s','full'), d.get('dec_solo_ms', d.get('full_ms')))" | tr '\n' ';'; echo; done
