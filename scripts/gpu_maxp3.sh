#!/bin/bash
# K-split cap sweep with the 3 x 8 KB ring
for MM in "2b 8" "2b 6" "2b 4" "7b 8" "7b 6" "7b 4"; do set -- $MM; echo "$1 maxP $2"; NOVA_GEMV_MAXP=$2 timeout 300 python scripts/dec_slice_probe.py --model $1 2>&1 | grep "^{" | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d.get('s','full'), d.get('dec_solo_ms', d.get('full_ms')))" | tr '\n' ';'; echo; done
