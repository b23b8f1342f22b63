#!/bin/bash
# Experiment: grouped-GEMM ring depths (MOESHARD_TC_VARIANT) on the bench workload.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
for v in ${VARIANTS:-0 2 5 6 7}; do
  MOESHARD_TC_VARIANT=$v timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/var_$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/var_$v.json')); k=d['kernels_us']
print('variant $v', round(d['ms_per_step']*1e3,1), 'us/step  up', k['gemm_up']['us'], 'down', k['gemm_down']['us'], 'skew', round(d['skewed']['ms_per_step']*1e3,1))"
done
