#!/bin/bash
# Eq. 5 readings on B200 (configs[1] 2B Poisson): adaptive SM_op x SM_min grid vs static 24 / serial
mkdir -p gpurun_out
timeout 2400 python scripts/policy_sweep.py --model 2b --trace poisson --rho 0.7 0.9 --seeds 3 --requests 96 \
  --sm-min 16 24 32 --sm-op 48 72 --static 24 --policies serial > gpurun_out/r2_policy.jsonl 2> gpurun_out/r2_policy.err
echo "rc=$?"; cat gpurun_out/r2_policy.jsonl | cut -c1-300; tail -2 gpurun_out/r2_policy.err
