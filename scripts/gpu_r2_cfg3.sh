#!/bin/bash
# configs[2] (7B, bursty GUI-agent trace, adaptive Pareto repartitioning) on the session-3 code
mkdir -p gpurun_out
timeout 2400 python bench.py --workload cfg3 > gpurun_out/r2_cfg3.json 2> gpurun_out/r2_cfg3.err; echo "bench rc=$?"
tail -3 gpurun_out/r2_cfg3.err
python - <<'P'
import json
d=json.load(open('gpurun_out/r2_cfg3.json'))
print(d['value'], d['req_per_s'], d['e2e']['value'], d['roofline'])
for r,c in d.get('compare',{}).items():
    print(r, {k:(v['max_ms'],v['req_per_s']) for k,v in c['policies'].items()})
print(d['stages_solo'])
print(d.get('plan'))
P
