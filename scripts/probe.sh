#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"push|reduce_part|wait_tok|rs_sig" -c 16 --csv python bench.py --transport p2p --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --encoder none --sustained 0 2>/dev/null | grep -E "push|reduce_part|wait_tok|rs_sig" | head -40 > gpurun_out/ncu_p2p.csv
wc -l gpurun_out/ncu_p2p.csv
