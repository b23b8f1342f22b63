#!/bin/bash
# Local helper: build here first (fail fast), then run the given command on the GPU box.
set -e
cd /root/repo
python paper_2503_08467_b200/_build.py > /dev/null
timeout ${GPU_TIMEOUT:-2400} /usr/local/graft/bin/gpurun --timeout ${GPU_LIMIT:-1500} -- "$@"
