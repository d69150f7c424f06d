#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2v1_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2v1_pytest.log
timeout 120 python __graft_entry__.py smoke 2>&1 | tail -1
timeout 1500 python bench.py > gpurun_out/r2v1_bench.json 2> gpurun_out/r2v1_bench.err; echo "bench rc=$?"
tail -3 gpurun_out/r2v1_bench.err
