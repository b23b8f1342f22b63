#!/bin/bash
# ncu of the narrow-shard FFN kernels (on-chip-H expert MLP vs the two-phase kernel)
# at the G = 8 per-rank shapes of C2 and C5 (flag 0x40000 = MOESHARD_FLAG_ONCHIP_H). usage: bash scripts/prof_mlp.sh [out-prefix]
OUT=${1:-gpurun_out/prof_mlp}
python -c "import __graft_entry__ as g; g.build()" > /dev/null
M='--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,launch__grid_size'
for shape in "8192 768 384 64" "32768 1024 512 128"; do
  for fl in 0x40000 0; do
    echo "== $shape flags=$fl"
    ncu $M --clock-control none -k regex:"tc_expert|tc_moe" -s 3 -c 2 python scripts/prof_shape.py $shape $fl 2>&1 | grep -E "^  [a-z]|duration|dram__bytes|tensor|dram_thr|grid_size" | head -14
  done
done
ncu --set full --clock-control none --import-source on -k regex:tc_expert -s 3 -c 1 -o ${OUT}_c2g8 python scripts/prof_shape.py 8192 768 384 64 > /dev/null 2>&1
echo done
