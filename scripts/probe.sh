#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_p2p_multiprocess.py -m gpu -x -q --timeout 200 -p no:cacheprovider > gpurun_out/pytest_quick.log 2>&1; rc=$?; echo "pytest rc=$rc"; tail -30 gpurun_out/pytest_quick.log | grep -E "passed|failed|Error|assert|error" | head -20
