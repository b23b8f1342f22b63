#!/bin/bash
# Round measurement script (run under gpurun): tests, bench line, ncu launch list, ncu full capture.
# usage: bash scripts/gpu_bench_profile.sh <tag> [full-kernel-regex] [skip-tests]
TAG=${1:-r02}
KRE=${2:-tc_moe_ffn}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
if [ -z "$3" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q --timeout 600 -p no:cacheprovider -rA > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_$TAG.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log
fi
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
tail -2 gpurun_out/bench_$TAG.err
OURS='regex:router|group_|tc_grouped|tc_moe|expert_mlp|simt_grouped|transpose|push_|reduce_'
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "$OURS" -c 200 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --encoder none --sustained 0 > /dev/null 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$KRE" -s 6 -c 1 -o gpurun_out/prof_$TAG python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e --encoder none --sustained 0 > gpurun_out/ncu_full_$TAG.log 2>&1; echo "ncu full rc=$?"
