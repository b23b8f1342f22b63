#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q --timeout 120 -p no:cacheprovider > gpurun_out/pytest_quick.log 2>&1; rc=$?; echo "pytest rc=$rc"; tail -2 gpurun_out/pytest_quick.log
[ $rc -ne 0 ] && exit 1
run() { timeout 200 python scripts/shape_probe.py $SHAPE 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', {r: (d[r]['step_us'], d[r]['phases_us']['gemm_up']) for r in ('uniform','zipf')})"; }
for rep in 1 2; do
for sh in "64 768 3072 8192 1" "64 768 3072 8192 8" "128 1024 4096 32768 8" "128 768 3072 16384 4"; do
  SHAPE="$sh" run "[$sh] light"; SHAPE="$sh" MOESHARD_LIGHT_RELEASE=0 run "[$sh] fence"
done
done
