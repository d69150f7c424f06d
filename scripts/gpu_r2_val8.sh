#!/bin/bash
# Full validation after the decode changes (qkv / o on gemv_umma, ln1 fold, attention ring by partition)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2v8_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2v8_pytest.log
timeout 120 python __graft_entry__.py smoke 2>&1 | tail -1
timeout 1800 python bench.py > gpurun_out/r2v8_bench.json 2> gpurun_out/r2v8_bench.err; echo "bench rc=$?"
tail -2 gpurun_out/r2v8_bench.err
python - <<'P'
import json
d=json.load(open('gpurun_out/r2v8_bench.json'))
print(d['value'], d['req_per_s'], d['e2e']['value'], d['roofline'])
for r,c in d.get('compare',{}).items():
    print(r, {k:(v['max_ms'],v['req_per_s']) for k,v in c['policies'].items()})
print(d['stages_solo'])
print(d.get('stages_solo_cfg3_7b'))
print(d.get('plan'))
P
python - <<'P'
import json
d=json.load(open('gpurun_out/r2v8_bench.json'))
print({k: v for k, v in d['kernels'].items()})
P
