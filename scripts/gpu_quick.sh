#!/bin/bash
# quick loop: build, GPU parity tests, variant timings
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_quick.log
VARIANTS="${VARIANTS:-0 2}" bash scripts/gemm_variants.sh 2>&1 | grep variant
