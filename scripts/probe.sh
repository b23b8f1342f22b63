#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 400 -p no:cacheprovider -k "fp32_validation_mode_c2 or staged_forward" -s 2>&1 | tail -8
