#!/bin/bash
# the bench command's ncu launch list over the timed region, with decode kernels visible: partitions as
# SM-budget-limited grids on primary-context streams (NOVA_BENCH_GREEN=0) -- ncu does not profile kernels in
# green contexts; shares only, never a bench number
mkdir -p gpurun_out
NOVA_BENCH_GREEN=0 NOVA_PROFILER_RANGE=1 timeout 1500 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/rf_launches_bench_ng.csv python bench.py --skip-profile --requests 6 --steps 1 --warmup 1 --no-compare --no-solo-7b > gpurun_out/rf_bench_ncu_ng.log 2>&1
echo "ncu rc=$?"
python scripts/ncu_summary.py --launches gpurun_out/rf_launches_bench_ng.csv --out gpurun_out/rf_launches_bench_ng.json > /dev/null 2>&1
python - <<'P'
import json
d = json.load(open('gpurun_out/rf_launches_bench_ng.json'))
tot = sum(x['launches'] for x in d['launches'])
print('launches', tot)
for x in d['launches'][:16]:
    print(x['kernel'][:60], x['launches'], round(x['total_us']), x['share'])
P
tail -2 gpurun_out/rf_bench_ncu_ng.log
