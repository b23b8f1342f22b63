#!/bin/bash
# A/B on one box: each argument is an env assignment string, e.g. "MOESHARD_TC_VARIANT=20"
mkdir -p gpurun_out
i=0
for envs in "$@"; do
  env $envs python bench.py --steps ${STEPS:-300} --no-cpu-baseline --no-e2e --encoder none > gpurun_out/abe_$i.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/abe_$i.json')); k=d['kernels_us']
ffn = k.get('expert_ffn', k.get('gemm_up'))
print('[$envs]', round(d['ms_per_step']*1e3,1), 'us/step  skew', round(d['skewed']['ms_per_step']*1e3,1), ' ffn', ffn['us'])"
  i=$((i+1))
done
