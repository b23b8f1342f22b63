#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_quick.log | grep -v "^$"
run() { timeout 300 python scripts/shape_probe.py 64 768 3072 8192 ${G:-1} 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', {r: (d[r]['step_us'], d[r]['phases_us']) for r in ('uniform','zipf')})"; }
for rep in 1 2; do
for fl in 0 256; do MOESHARD_FLAGS=$fl run "flags $fl"; done
done
for G in 2 8; do for fl in 0 256; do G=$G MOESHARD_FLAGS=$fl run "G$G flags $fl"; done; done
