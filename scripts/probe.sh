#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1200 python -m pytest tests -m gpu -q --timeout 400 -p no:cacheprovider > gpurun_out/pytest_all.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_all.log
timeout 600 python bench.py > gpurun_out/bench_r01g.json 2> gpurun_out/bench_r01g.err; echo "bench rc=$?"
timeout 900 python bench.py --config c5 --steps 100 --warmup 10 --no-e2e --encoder c5 --sustained 0 > gpurun_out/bench_c5g.json 2> gpurun_out/bench_c5g.err; echo "c5 rc=$?"
timeout 600 python bench.py --config c3 --steps 200 --warmup 20 --no-e2e --encoder none --sustained 0 > gpurun_out/bench_c3g.json 2> gpurun_out/bench_c3g.err; echo "c3 rc=$?"
