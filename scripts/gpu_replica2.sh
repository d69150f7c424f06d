#!/bin/bash
# functional check of bench.py's replica path (torchrun, 2 ranks) on a one-GPU box
mkdir -p gpurun_out
export NOVA_BENCH_SAME_GPU=1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 2 --steps 1 --warmup 1 --requests 8 --quick --no-compare > gpurun_out/replica2.out 2> gpurun_out/replica2.err
echo "rc=$?"; tail -c 800 gpurun_out/replica2.out; grep -i "error\|Traceback" gpurun_out/replica2.err | head -5
