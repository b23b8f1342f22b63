#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
run() { timeout 300 python scripts/shape_probe.py 64 768 3072 8192 ${G:-1} 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', {r: (d[r]['step_us'], d[r]['phases_us']['gemm_up']) for r in ('uniform','zipf')})"; }
for pl in 0 32 64 79; do MOESHARD_L2_PERSIST_MB=$pl run "persist $pl"; done
for gd in 3 4 5; do MOESHARD_FLAGS=64 MOESHARD_GATHER_DEPTH=$gd MOESHARD_L2_PERSIST_MB=48 run "cpasync depth $gd"; done
G=8 MOESHARD_FLAGS=64 MOESHARD_GATHER_DEPTH=5 MOESHARD_L2_PERSIST_MB=48 run "G8 cpasync depth 5"
