#!/bin/bash
L=paper_2509_21301_b200
cp $L/libnova_new.so $L/libnova.so
timeout 300 python -m pytest tests/test_gpu_gemv_umma.py -x -q 2>&1 | tail -3
for ck in 2 4 8 24; do
  echo "ckmin=$ck"
  NOVA_UMMA_CKMIN=$ck timeout 300 python scripts/ubench.py --only 2b_gu --iters 20 2>&1 | grep '"B": 2'
  NOVA_UMMA_CKMIN=$ck timeout 300 python scripts/ubench.py --only 2b_lm --iters 10 2>&1 | grep '"B": 2'
done
cp $L/libnova_old.so $L/libnova.so
echo old; timeout 300 python scripts/ubench.py --only 2b_gu --iters 20 2>&1 | grep '"B": 2'
timeout 300 ncu --set full --clock-control none -k regex:gemv_umma -s 5 -c 1 -o gpurun_out/r2_sk_old_lm python scripts/ubench.py --only 2b_lm --iters 2 > /dev/null 2>&1
cp $L/libnova_new.so $L/libnova.so
timeout 300 ncu --set full --clock-control none -k regex:gemv_umma -s 5 -c 1 -o gpurun_out/r2_sk_new_lm python scripts/ubench.py --only 2b_lm --iters 2 > /dev/null 2>&1
ls gpurun_out/
