#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q --timeout 300 -p no:cacheprovider -k "natural or c2_full or c3 or tcgen05_parity" > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_quick.log | grep -E "passed|failed|Error|assert"
for r in 0 1; do MOESHARD_ROUTER_ROT=$r MOESHARD_ROUTER_TIMING=1 timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --encoder none --sustained 0 2>&1 | grep "router cta" | head -4; done
b() { timeout 300 python bench.py --steps 300 --warmup 20 --no-cpu-baseline --no-e2e --encoder none --sustained 0 > gpurun_out/ab.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/ab.json')); k=d['kernels_us']; print('$1 step', round(d['ms_per_step']*1e3,2), 'skew', round(d['skewed']['ms_per_step']*1e3,2), d['clocks']['sm_mhz'], 'router', k['router']['us'], 'grouping', k['grouping']['us'], 'ffn', k['expert_ffn']['us'])"; }
for rep in 1 2; do
MOESHARD_ROUTER_ROT=0 b "rot0"
b "rot1"
done
run() { timeout 300 python scripts/shape_probe.py 64 768 3072 8192 ${G:-1} 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', {r: (d[r]['step_us'], d[r]['phases_us']) for r in ('uniform','zipf')})"; }
G=8 run "G8 fused"
G=8 MOESHARD_FLAGS=4 run "G8 unfused"
G=4 run "G4 fused"
G=4 MOESHARD_FLAGS=4 run "G4 unfused"
