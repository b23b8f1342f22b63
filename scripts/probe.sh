#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 120 -p no:cacheprovider -k "p2p" > gpurun_out/pytest_p2p.log 2>&1; echo "p2p pytest rc=$?"; tail -30 gpurun_out/pytest_p2p.log | grep -E "passed|failed|Error|assert" 
for rep in 1 2; do
for fl in 0 128; do
  MOESHARD_FLAGS=$fl timeout 300 python bench.py --steps 300 --warmup 20 --no-cpu-baseline --no-e2e --encoder none --sustained 0 > gpurun_out/ab_$fl.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/ab_$fl.json')); print('flags $fl step', round(d['ms_per_step']*1e3,2), 'skew', round(d['skewed']['ms_per_step']*1e3,2), d['clocks'])"
done
done
