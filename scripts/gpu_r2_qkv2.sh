#!/bin/bash
# qkv on gemv_umma with the 2-deep fold (ring >= 1): decode splits, then the default bench with o on umma.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_gemv_umma.py -q -x 2>&1 | tail -1
for v in "NOVA_DEC_TMA=30"; do
  env $v timeout 300 python scripts/dec_splits.py --model 2b --B 2 16 --splits 0 24 32 48 72 2>&1 | grep '^{'
  env $v timeout 300 python scripts/dec_splits.py --model 7b --B 2 16 --splits 0 24 32 48 72 2>&1 | grep '^{'
done
NOVA_DEC_TMA=30 timeout 1800 python bench.py > gpurun_out/r2q2_bench.json 2> gpurun_out/r2q2_bench.err; echo "bench rc=$?"
tail -2 gpurun_out/r2q2_bench.err
python - <<'P'
import json
d=json.load(open('gpurun_out/r2q2_bench.json'))
print(d['value'], d['req_per_s'], d['e2e']['value'], d['roofline'])
for r,c in d.get('compare',{}).items():
    print(r, {k:(v['max_ms'],v['req_per_s']) for k,v in c['policies'].items()})
print(d['stages_solo'])
print(d.get('stages_solo_cfg3_7b'))
P
