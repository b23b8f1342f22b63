#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
MOESHARD_PAIR_DOWN=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q --timeout 200 -p no:cacheprovider > gpurun_out/pytest_pair.log 2>&1; rc=$?; echo "pytest(pair) rc=$rc"; tail -3 gpurun_out/pytest_pair.log | grep -E "passed|failed|Error"
[ $rc -ne 0 ] && { grep -E "Error|assert" gpurun_out/pytest_pair.log | head; exit 1; }
run() { timeout 200 python scripts/shape_probe.py $SHAPE 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', {r: (d[r]['step_us'], d[r]['phases_us']['gemm_up']) for r in ('uniform','zipf')})"; }
for rep in 1 2; do
for sh in "64 768 3072 8192 1" "128 768 3072 16384 1" "128 1024 4096 32768 1 60" "64 768 3072 8192 8"; do
  SHAPE="$sh" run "[$sh] base"; SHAPE="$sh" MOESHARD_PAIR_DOWN=1 run "[$sh] pair"
done
done
