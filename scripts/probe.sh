#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_p2p_multiprocess.py -m gpu -x -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_quick.log 2>&1; rc=$?; echo "pytest rc=$rc"; tail -2 gpurun_out/pytest_quick.log
[ $rc -ne 0 ] && { grep -E "Error|assert" gpurun_out/pytest_quick.log | head; exit 1; }
b() { timeout 300 python bench.py --steps 300 --warmup 20 --no-cpu-baseline --no-e2e --encoder none --sustained 0 > gpurun_out/ab.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/ab.json')); print('$1 step', round(d['ms_per_step']*1e3,2), 'skew', d['skewed']['skew_over_uniform_time'], d['clocks']['sm_mhz'])"; }
for rep in 1 2 3; do
b "early"
MOESHARD_EARLY_TABLES=0 b "late"
done
run() { timeout 200 python scripts/shape_probe.py $SHAPE 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', {r: (d[r]['step_us'], d[r]['phases_us']['gemm_up']) for r in ('uniform','zipf')})"; }
for sh in "64 768 3072 8192 8" "128 1024 4096 32768 8" "128 768 3072 16384 1"; do
  SHAPE="$sh" run "[$sh] early"; SHAPE="$sh" MOESHARD_EARLY_TABLES=0 run "[$sh] late"
done
