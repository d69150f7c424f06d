#!/bin/bash
for V in base sleep base sleep; do cp build/var/libnova_$V.so paper_2509_21301_b200/libnova.so; echo "$V"; timeout 300 python scripts/dec_slice_probe.py --model 2b 2>&1 | grep "^{" | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d.get('s','full'), d.get('dec_solo_ms', d.get('full_ms')))" | tr '\n' ';'; echo; done
cp build/var/libnova_sleep.so paper_2509_21301_b200/libnova.so
