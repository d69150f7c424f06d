#!/bin/bash
# why is the causal key split slow? ncu full capture of the split and unsplit causal FMHA (2B prefill shape)
mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on"
for c in 0 1; do
  NOVA_FMHA_CSPLIT=$c timeout 300 $NCU -k regex:fmha4 -s 2 -c 1 -o gpurun_out/cs_fmha_$c -f python scripts/attn_one.py 1286 12 2 128 1 4 > gpurun_out/cs_ncu_$c.log 2>&1
  echo "ncu c=$c rc=$?"
  ncu -i gpurun_out/cs_fmha_$c.ncu-rep --page details --csv 2>/dev/null | grep -E '"Duration"|"Warp Cycles Per Issued|Stall|"Achieved Occupancy"|Registers Per|Local Memory|"Elapsed Cycles"|DRAM Throughput|"L2 Hit' | head -30
done
