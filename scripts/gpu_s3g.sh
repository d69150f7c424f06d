#!/bin/bash
# session-3 final validation: all GPU tests, smoke, kernel micro-bench, bench
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python scripts/kbench.py > gpurun_out/kbench_s3g.jsonl 2>&1; wc -l gpurun_out/kbench_s3g.jsonl
timeout 300 python scripts/pass_profile.py --stage all > gpurun_out/pass_s3g.jsonl 2>/dev/null
for B in 1 4 8 16; do timeout 120 python scripts/pass_profile.py --stage dec --B $B 2>/dev/null; done >> gpurun_out/pass_s3g.jsonl
cat gpurun_out/pass_s3g.jsonl
timeout 1500 python bench.py --out gpurun_out/bench_s3g.json 2>gpurun_out/bench_s3g.err | tail -c 200; tail -3 gpurun_out/bench_s3g.err
timeout 300 python bench.py --impl reference --steps 1 --warmup 1 2>&1 | tail -c 300
