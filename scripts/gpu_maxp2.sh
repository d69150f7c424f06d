#!/bin/bash
for MM in "7b 8" "7b 12" "2b 6" "2b 12"; do set -- $MM; echo "$1 maxP $2"; NOVA_GEMV_MAXP=$2 timeout 300 python scripts/dec_slice_probe.py --model $1 2>&1 | grep "^{" | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d.get('s','full'), d.get('dec_solo_ms', d.get('full_ms')))" | tr '\n' ';'; echo; done
