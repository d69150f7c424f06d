#!/bin/bash
# session-3 checkpoint: full GPU tests, smoke, per-stage solo passes + launch lists + full ncu
# captures of the hot kernels, default bench, bench launch list
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
bash scripts/gpu_prof.sh > gpurun_out/prof.log 2>&1; tail -3 gpurun_out/prof.log
timeout 1500 python bench.py --out gpurun_out/bench_s3b.json 2>gpurun_out/bench_s3b.err | tail -c 600; tail -3 gpurun_out/bench_s3b.err
NOVA_PROFILER_RANGE=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --skip-profile --requests 4 --steps 1 --warmup 1 --no-compare > gpurun_out/bench_ncu.log 2>&1
python scripts/ncu_summary.py --launches gpurun_out/launches_bench.csv --out gpurun_out/launches_bench.json > /dev/null 2>&1; ls gpurun_out
