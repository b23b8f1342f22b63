#!/bin/bash
# A/B in one box: bench step time for several MOESHARD_FLAGS values (same process image, same GPU)
mkdir -p gpurun_out
for f in ${FLAGSETS:-0 8}; do
  MOESHARD_FLAGS=$f python bench.py --steps ${STEPS:-300} --no-cpu-baseline --no-e2e > gpurun_out/ab_$f.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/ab_$f.json')); k=d['kernels_us']
print('flags $f:', round(d['ms_per_step']*1e3,1), 'us/step  skew', round(d['skewed']['ms_per_step']*1e3,1), ' router', k['router']['us'], 'grouping', k['grouping']['us'], 'ffn', k['gemm_up']['us'])"
done
