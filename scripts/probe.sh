#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_quick.log 2>&1; rc=$?; echo "pytest rc=$rc"; tail -2 gpurun_out/pytest_quick.log
[ $rc -ne 0 ] && { grep -E "Error|assert" gpurun_out/pytest_quick.log | head; exit 1; }
b() { timeout 300 python bench.py --steps 300 --warmup 20 --no-cpu-baseline --no-e2e --encoder none --sustained 0 > gpurun_out/ab.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/ab.json')); print('$1 step', round(d['ms_per_step']*1e3,2), 'skew', d['skewed']['skew_over_uniform_time'], d['clocks']['sm_mhz'], d['gpu_launches'])"; }
for rep in 1 2 3; do
b "router-scan"
MOESHARD_ROUTER_SCAN=0 b "scan-launch"
done
