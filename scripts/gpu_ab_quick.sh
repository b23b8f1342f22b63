#!/bin/bash
# build, GPU tests, then bench A/B of MOESHARD_FLAGS values given in $AB (default "0 32")
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_quick.log | grep -v "^$"
for rep in 1 2; do
for f in ${AB:-0 32}; do
  MOESHARD_FLAGS=$f timeout 300 python bench.py --steps 300 --warmup 20 --no-cpu-baseline --no-e2e --encoder none --sustained 0 ${BENCH_ARGS} > gpurun_out/ab_$f.json 2>/dev/null
  python - $f <<'PY'
import json, sys
d = json.load(open(f"gpurun_out/ab_{sys.argv[1]}.json"))
k = d["kernels_us"]
print(f"flags={sys.argv[1]:>3} step {d['ms_per_step']*1e3:7.2f} us  skew {d['skewed']['ms_per_step']*1e3:7.2f} us  " +
      " ".join(f"{n}={v['us']:.1f}" for n, v in k.items()), d["clocks"]["sm_mhz"])
PY
done
done
