#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q 2>&1 | tail -3
timeout 100 python scripts/kbench.py --only dattn
timeout 300 compute-sanitizer --tool memcheck --print-limit 5 python -m pytest tests/test_gpu_kernels.py -x -q -k "gemv_tma or decode_attention" 2>&1 | tail -8
NOVA_PROFILER_RANGE=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --skip-profile --requests 4 --steps 1 --warmup 1 --no-compare > gpurun_out/bench_ncu.log 2>&1
grep -c gemv gpurun_out/launches.csv; grep ERROR gpurun_out/launches.csv | head -3
timeout 900 python bench.py --requests 32 --steps 2 --warmup 1 --out gpurun_out/bench5.json 2>gpurun_out/bench5.err; tail -3 gpurun_out/bench5.err
