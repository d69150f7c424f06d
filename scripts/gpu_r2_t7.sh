#!/bin/bash
for dbg in 4 12 20 28; do for s in 32; do
NOVA_DEC_FUSED_DBGX=$dbg timeout 300 python scripts/fd_timeline.py --model 2b --s $s 2>&1 | grep "^{" | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('dbg=$dbg', 's=$s', d['ms'], json.dumps(d['last_layer_span_us']))"
done; done
