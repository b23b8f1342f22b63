#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python -m pytest tests/test_p2p_multiprocess.py tests/test_bench_contract.py -m gpu -x -q --timeout 400 -p no:cacheprovider 2>&1 | tail -30
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"
