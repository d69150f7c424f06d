#!/bin/bash
cat > /tmp/sp.py <<'PY'
import sys, json; sys.path.insert(0, '.')
import bench as BN
from synth import Q2B, Q7B
sh = Q2B if sys.argv[1] == '2b' else Q7B
eng = BN.build_engine(sh, 0)
eng.time_pass(2, 0, B=2, ctx=1334, iters=3)
out = {}
for s in [0, 24, 32, 48, 64]:
    out[s] = round(eng.time_pass(2, s, B=2, ctx=1334, iters=8)[0], 3)
print(json.dumps(out))
PY
for m in 0 20 28 30 16; do echo -n "mask=$m 2b "; NOVA_UMMA_MASK=$m timeout 300 python /tmp/sp.py 2b 2>&1 | tail -1; done
for m in 0 28 30; do echo -n "mask=$m 7b "; NOVA_UMMA_MASK=$m timeout 300 python /tmp/sp.py 7b 2>&1 | tail -1; done
