#!/bin/bash
# bench command's launch list with profiling from the start (green-context decode kernels included?)
mkdir -p gpurun_out
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/rf_launches_bench_all.csv python bench.py --skip-profile --requests 4 --steps 1 --warmup 1 --no-compare --no-solo-7b > gpurun_out/rf_bench_ncu_all.log 2>&1
echo "ncu rc=$?"
python scripts/ncu_summary.py --launches gpurun_out/rf_launches_bench_all.csv --out gpurun_out/rf_launches_bench_all.json > /dev/null 2>&1
python - <<'P'
import json
d = json.load(open('gpurun_out/rf_launches_bench_all.json'))
for x in d['launches'][:14]:
    print(x['kernel'][:60], x['launches'], round(x['total_us']), x['share'])
P
tail -3 gpurun_out/rf_bench_ncu_all.log
