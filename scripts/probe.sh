#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
for pol in first normal; do
MOESHARD_SIBLING_POLICY=$pol timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k "regex:tc_moe_ffn" -s 3 -c 2 --csv python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --encoder none --sustained 0 2>/dev/null | grep -E "tc_moe" | awk -F'","' -v p=$pol '{print p, $(NF-2), $NF}'
MOESHARD_SIBLING_POLICY=$pol timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k "regex:tc_moe_ffn" -s 3 -c 2 --csv python scripts/shape_probe.py 64 768 3072 8192 1 3 2>/dev/null | grep -E "tc_moe" | tail -6 | awk -F'","' -v p=$pol '{print "c2probe", p, $(NF-2), $NF}'
done
