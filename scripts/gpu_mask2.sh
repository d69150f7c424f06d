#!/bin/bash
for M in 28 29 30 31; do echo "mask $M"; NOVA_DEC_TMA=$M timeout 300 python scripts/dec_slice_probe.py --model 2b 2>&1 | grep "^{" | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d.get('s','full'), d.get('dec_solo_ms', d.get('full_ms')), d.get('dec_corun_vit_ms',''))" | tr '\n' ';'; echo; done
for M in 28 31; do echo "7b mask $M"; NOVA_DEC_TMA=$M timeout 300 python scripts/dec_slice_probe.py --model 7b 2>&1 | grep "^{" | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d.get('s','full'), d.get('dec_solo_ms', d.get('full_ms')), d.get('dec_corun_vit_ms',''))" | tr '\n' ';'; echo; done
