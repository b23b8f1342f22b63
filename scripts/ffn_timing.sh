#!/bin/bash
mkdir -p gpurun_out
MOESHARD_TC_VARIANT=21 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --encoder none 2>&1 | grep "ffn c" > gpurun_out/ffn_timing.txt
python - <<'PY'
import re, statistics as st
lines = open('gpurun_out/ffn_timing.txt').read().splitlines()
runs = [lines[i:i+74] for i in range(0, len(lines), 74)]
for i, run in enumerate(runs[:9]):
    if len(run) != 74: continue
    rows=[tuple(int(x) for x in re.search(r'c(\d+)\] up (\d+) dn (\d+) kb (\d+) total (\d+) first_down (\d+) waitA (\d+) waitB (\d+) waitT (\d+)', l).groups()) for l in run]
    tot=[r[4] for r in rows]; busy=[r[4]-r[6]-r[7]-r[8] for r in rows]
    print(f"run{i}: total max {max(tot)} mean {st.mean(tot):.0f} min {min(tot)} | first_down {st.mean(r[5] for r in rows):.0f} | waitA {st.mean(r[6] for r in rows):.0f} waitB {st.mean(r[7] for r in rows):.0f} waitT {st.mean(r[8] for r in rows):.0f} busy {st.mean(busy):.0f}")
PY
