#!/bin/bash
# round 2: first run of the fused decode kernel (tiny parity, 2B/7B reduced depth, slices)
mkdir -p gpurun_out
timeout 300 python __graft_entry__.py smoke > gpurun_out/r2f1_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r2f1_smoke.log
timeout 600 python -m pytest tests/test_gpu_engine.py -x -q > gpurun_out/r2f1_engine.log 2>&1; echo "engine rc=$?"; tail -15 gpurun_out/r2f1_engine.log
timeout 300 python scripts/dec_slice_probe.py --model 2b > gpurun_out/r2f1_slice2b.jsonl 2>gpurun_out/r2f1_slice2b.err; echo "slice2b rc=$?"
timeout 300 python scripts/dec_slice_probe.py --model 7b > gpurun_out/r2f1_slice7b.jsonl 2>gpurun_out/r2f1_slice7b.err; echo "slice7b rc=$?"
cat gpurun_out/r2f1_slice2b.jsonl gpurun_out/r2f1_slice7b.jsonl | head -40
tail -3 gpurun_out/r2f1_slice2b.err
