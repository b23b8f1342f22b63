#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
run() { timeout 200 python scripts/shape_probe.py $SHAPE 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', {r: (d[r]['step_us'], d[r]['phases_us']['gemm_up']) for r in ('uniform','zipf')})"; }
for rep in 1 2; do
for sh in "64 768 3072 8192 1" "128 768 3072 16384 1" "64 768 3072 8192 8"; do
  for pl in 48 64 79; do SHAPE="$sh" MOESHARD_L2_PERSIST_MB=$pl run "[$sh] persist $pl"; done
done
done
