#!/bin/bash
timeout 300 python tests/dbg_fused.py 0 2>&1 | grep -a stop
for pf in 0 48; do for s in 0 32; do
NOVA_DEC_PF_MB=$pf timeout 300 python scripts/fd_timeline.py --model 2b --s $s 2>&1 | grep "^{" | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('pf=$pf', 's=$s', d['ms'], json.dumps(d['last_layer_milestones_us']), json.dumps(d['last_layer_span_us']))"
done; done
