#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
OURS='regex:router_tc|group_|tc_moe_ffn'
timeout 900 ncu --set full --clock-control none --import-source on -k "$OURS" -s 8 -c 4 -o gpurun_out/prof_final_c2 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e --encoder none --sustained 0 > gpurun_out/ncu_final_c2.log 2>&1; echo "ncu c2 rc=$?"
timeout 900 ncu --set full --clock-control none -k "regex:tc_moe_ffn" -s 2 -c 1 -o gpurun_out/prof_final_c5 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --encoder none --sustained 0 > gpurun_out/ncu_final_c5.log 2>&1; echo "ncu c5 rc=$?"
