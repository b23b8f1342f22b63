#!/bin/bash
mkdir -p gpurun_out
for mb in ${MBS:-0 20 40 60 80}; do
  MOESHARD_L2_PREFETCH_MB=$mb python bench.py --steps 300 --no-cpu-baseline --no-e2e > gpurun_out/pf_$mb.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/pf_$mb.json')); k=d['kernels_us']
print('prefetch $mb MB:', round(d['ms_per_step']*1e3,1), 'us/step  skew', round(d['skewed']['ms_per_step']*1e3,1), ' router', k['router']['us'], 'ffn', k['gemm_up']['us'])"
done
