#!/bin/bash
mkdir -p gpurun_out
timeout 600 python scripts/dbg_fused.py off 0 1 3 4 5 6 8 9 10 11 > gpurun_out/r2d1_bisect.log 2>&1; echo "bisect rc=$?"
grep stop gpurun_out/r2d1_bisect.log; grep -i error gpurun_out/r2d1_bisect.log | head -5
cat > /tmp/dec2b.py <<'PY'
import sys; sys.path.insert(0, '.')
import bench as BN
from synth import Q2B
sh = Q2B
import dataclasses
sh = dataclasses.replace(Q2B, llm_layers=2, vit_depth=1)
eng = BN.build_engine(sh, 0)
print(eng.time_pass(2, 0, B=2, ctx=300, iters=1))
PY
timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --print-limit 10 python /tmp/dec2b.py > gpurun_out/r2d1_memcheck.log 2>&1; echo "memcheck rc=$?"
head -60 gpurun_out/r2d1_memcheck.log
