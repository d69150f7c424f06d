#!/bin/bash
# decode GEMV ring geometry sweep (build/var/libnova_{base,v1,v2,v3}.so, see gemv_tma.cu GEMV_* macros)
for M in 2b 7b; do for V in v3 v4 v5 v6; do cp build/var/libnova_$V.so paper_2509_21301_b200/libnova.so; echo "$M $V"; timeout 300 python scripts/dec_slice_probe.py --model $M 2>&1 | grep "^{" | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d.get('s','full'), d.get('dec_solo_ms', d.get('full_ms')))" | tr '\n' ';'; echo; done; done
cp build/var/libnova_base.so paper_2509_21301_b200/libnova.so
