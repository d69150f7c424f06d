#!/bin/bash
# Per-stage solo pass timings + ncu launch lists + one full capture per hot kernel class.
mkdir -p gpurun_out
P="python scripts/pass_profile.py"
timeout 300 $P --stage all > gpurun_out/pass.jsonl 2>gpurun_out/pass.err; cat gpurun_out/pass.jsonl; tail -2 gpurun_out/pass.err
for B in 1 4 8 16; do timeout 120 $P --stage dec --B $B 2>/dev/null; done | tee -a gpurun_out/pass.jsonl
for st in dec vit pre; do
  timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launch_$st.csv $P --stage $st --profile > /dev/null 2>&1
  python scripts/ncu_summary.py --launches gpurun_out/launch_$st.csv --out gpurun_out/launch_$st.json > /dev/null
done
NCU="ncu --profile-from-start off --set full --clock-control none --import-source on"
timeout 600 $NCU -k regex:gemv_kernel -c 3 -o gpurun_out/ncu_dec_gemv -f $P --stage dec --profile > /dev/null 2>&1
timeout 600 $NCU -k regex:gemv_tma -c 1 -o gpurun_out/ncu_dec_gemv_tma -f $P --stage dec --profile > /dev/null 2>&1
timeout 600 $NCU -k regex:decode_attn -c 2 -o gpurun_out/ncu_dec_attn -f $P --stage dec --profile > /dev/null 2>&1
timeout 600 $NCU -k regex:fmha -c 1 -o gpurun_out/ncu_vit_fmha -f $P --stage vit --profile > /dev/null 2>&1
timeout 600 $NCU -k regex:gemm_tc -c 5 -o gpurun_out/ncu_vit_gemm -f $P --stage vit --profile > /dev/null 2>&1
ls gpurun_out
