#!/bin/bash
# Full measurement pass (run under gpurun): GPU tests + smoke, default bench line, ncu launch
# list of the bench step, one ncu --set full capture of every library kernel of the step,
# per-rank sweep and per-rank invariance. Outputs in gpurun_out/<tag>_*.
TAG=${1:-r02c}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 600 -p no:cacheprovider -rA > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
OURS='regex:router|group_|tc_grouped|tc_moe|expert_mlp|simt_grouped|transpose|push_|reduce_'
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "$OURS" -c 200 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --encoder none --sustained 0 > /dev/null 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k "$OURS" -s 24 -c 4 -o gpurun_out/${TAG}_prof python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e --encoder none --sustained 0 > gpurun_out/${TAG}_ncu_full.log 2>&1; echo "ncu full rc=$?"
timeout 900 python scripts/rank_sweep.py > gpurun_out/${TAG}_rank_sweep.json 2> gpurun_out/${TAG}_rank_sweep.err; echo "rank_sweep rc=$?"
timeout 900 python scripts/invariance.py > gpurun_out/${TAG}_invariance.json 2> gpurun_out/${TAG}_invariance.err; echo "invariance rc=$?"
