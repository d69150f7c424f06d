#!/bin/bash
# Round-2 session-3 validation of HEAD: GPU tests, smoke, default bench, launch list.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2v3_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2v3_pytest.log
timeout 120 python __graft_entry__.py smoke 2>&1 | tail -1
timeout 1800 python bench.py > gpurun_out/r2v3_bench.json 2> gpurun_out/r2v3_bench.err; echo "bench rc=$?"
tail -2 gpurun_out/r2v3_bench.err
