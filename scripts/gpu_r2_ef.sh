#!/bin/bash
# L2 evict-first on the decode weight stream: co-run curves + timed serving replay, EF off vs on
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_gemv_umma.py -q -x 2>&1 | tail -1
for ef in 0 1; do
  NOVA_UMMA_EF=$ef timeout 900 python bench.py --no-compare --no-solo-7b --compare-rho 0.9 > gpurun_out/ef$ef.json 2> gpurun_out/ef$ef.err
  python - $ef <<'P'
import json, sys
d = json.load(open(f'gpurun_out/ef{sys.argv[1]}.json'))
c = d['curves']
print('EF', sys.argv[1], 'value', d['value'], 'rps', d['req_per_s'], 'vit_pass', round(d['stages']['vit_pass']['ms_per_launch'], 2),
      'pre_pass', round(d['stages']['pre_pass']['ms_per_launch'], 2), 'dec_pass', round(d['stages']['dec_pass']['ms_per_launch'], 3))
print(' t_v', c['t_v_ms']); print(' t_p', c['t_p_ms']); print(' t_d_dv', c['t_d_dv_ms'])
P
done
