#!/bin/bash
cat > /tmp/dec2b.py <<'PY'
import sys, dataclasses; sys.path.insert(0, '.')
import bench as BN
from synth import Q2B, Q7B
sh = dataclasses.replace(Q2B if sys.argv[1] == "2b" else Q7B, llm_layers=2, vit_depth=1)
eng = BN.build_engine(sh, 0)
print(eng.time_pass(2, 0, B=int(sys.argv[2]), ctx=int(sys.argv[3]), iters=1))
PY
timeout 300 python /tmp/dec2b.py 2b 2 1334 2>&1 | tail -1
timeout 300 python /tmp/dec2b.py 2b 1 20 2>&1 | tail -1
timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --print-limit 6 python /tmp/dec2b.py 2b 2 1334 > gpurun_out/r2d4_memcheck.log 2>&1; echo "memcheck rc=$?"
grep -v "^=========     Host Frame\|^=========         \|^========= *$" gpurun_out/r2d4_memcheck.log | head -50
