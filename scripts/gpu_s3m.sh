#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1500 python bench.py --workload cfg3 --out gpurun_out/bench_s3m_cfg3.json 2>gpurun_out/bench_s3m.err | tail -c 150; echo; grep -i "stall\|error\|Traceback" gpurun_out/bench_s3m.err | head -3
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 2>&1 | tail -c 200
