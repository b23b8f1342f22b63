#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
run() { timeout 200 python scripts/shape_probe.py $SHAPE 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', {r: (d[r]['step_us'], d[r]['phases_us']['gemm_up']) for r in ('uniform','zipf')})"; }
# correctness of the experiment path first
MOESHARD_TC_VARIANT=20 MOESHARD_A256=1 timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q --timeout 120 -p no:cacheprovider -k "c2_full or tcgen05_parity" 2>&1 | tail -2
for rep in 1 2; do
for sh in "64 768 3072 8192 1" "64 768 3072 8192 8" "128 768 3072 16384 4"; do
  SHAPE="$sh" run "[$sh] default"; SHAPE="$sh" MOESHARD_TC_VARIANT=20 run "[$sh] ka2"; SHAPE="$sh" MOESHARD_TC_VARIANT=20 MOESHARD_A256=1 run "[$sh] ka2+a256"
done
done
