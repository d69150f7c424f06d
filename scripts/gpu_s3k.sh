#!/bin/bash
# session-3 final: tests, smoke, kernels, solo passes, ncu captures of the hot kernels, bench
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python scripts/kbench.py > gpurun_out/kbench_s3k.jsonl 2>&1; wc -l gpurun_out/kbench_s3k.jsonl
timeout 300 python scripts/pass_profile.py --stage all > gpurun_out/pass_s3k.jsonl 2>/dev/null
for B in 1 4 8 16; do timeout 120 python scripts/pass_profile.py --stage dec --B $B 2>/dev/null; done >> gpurun_out/pass_s3k.jsonl
cat gpurun_out/pass_s3k.jsonl
for st in dec vit pre; do
  timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launch_s3k_$st.csv python scripts/pass_profile.py --stage $st --profile > /dev/null 2>&1
  python scripts/ncu_summary.py --launches gpurun_out/launch_s3k_$st.csv --out gpurun_out/launch_s3k_$st.json > /dev/null
done
NCU="ncu --profile-from-start off --set full --clock-control none --import-source on"
timeout 600 $NCU -k regex:gemm_tc -c 5 -o gpurun_out/ncu_s3k_vit_gemm -f python scripts/pass_profile.py --stage vit --profile > /dev/null 2>&1
timeout 600 $NCU -k regex:fmha -c 1 -o gpurun_out/ncu_s3k_vit_fmha -f python scripts/pass_profile.py --stage vit --profile > /dev/null 2>&1
timeout 600 $NCU -k regex:gemv_tma -c 2 -o gpurun_out/ncu_s3k_dec_gemv -f python scripts/pass_profile.py --stage dec --profile > /dev/null 2>&1
timeout 1500 python bench.py --out gpurun_out/bench_s3k.json 2>gpurun_out/bench_s3k.err | tail -c 200; echo; grep -i "stall\|error\|Traceback" gpurun_out/bench_s3k.err | head -3
ls gpurun_out | wc -l
