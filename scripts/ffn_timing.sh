#!/bin/bash
# Per-cluster clock64 counters of the fused FFN kernel (MOESHARD_TC_VARIANT=21).
# Extra env (e.g. MOESHARD_FFN_SCHED=rr) is passed through; output tag = $TAG.
mkdir -p gpurun_out
TAG=${TAG:-x}
MOESHARD_TC_VARIANT=21 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --encoder none --sustained 0 2>&1 | grep "ffn c" > gpurun_out/ffn_timing_$TAG.txt
TAG=$TAG python - <<'PY'
import re, os, statistics as st
lines = open(f"gpurun_out/ffn_timing_{os.environ['TAG']}.txt").read().splitlines()
runs = [lines[i:i+74] for i in range(0, len(lines), 74)]
for i, run in enumerate(runs[:9]):
    if len(run) != 74: continue
    rows=[tuple(int(x) for x in re.search(r'c(\d+)\] up (\d+) dn (\d+) kb (\d+) total (\d+) first_down (\d+) waitA (\d+) waitB (\d+) waitT (\d+) g_entry (\d+) g_ready (\d+) g_end (\d+)', l).groups()) for l in run]
    ge=[r[9] for r in rows]; gr=[r[10] for r in rows]; gn=[r[11] for r in rows]; g0=min(ge)
    print(f"   globaltimer us: entry {0:.1f}..{(max(ge)-g0)/1e3:.1f} ready {(min(gr)-g0)/1e3:.1f}..{(max(gr)-g0)/1e3:.1f} mma-loop end {(min(gn)-g0)/1e3:.1f}..{(max(gn)-g0)/1e3:.1f}")
    tot=[r[4] for r in rows]; busy=[r[4]-r[6]-r[7]-r[8] for r in rows]; kb=[r[3] for r in rows]
    mk=sum(kb)/len(kb); mt=sum(tot)/len(tot)
    cov=sum((a-mk)*(b-mt) for a,b in zip(kb,tot))/len(kb)
    corr=cov/(st.pstdev(kb)*st.pstdev(tot)+1e-9)
    print(f"{os.environ['TAG']} run{i}: total max {max(tot)} mean {mt:.0f} min {min(tot)} | kb max {max(kb)} min {min(kb)} corr {corr:.2f} | first_down {st.mean(r[5] for r in rows):.0f} | waitA {st.mean(r[6] for r in rows):.0f} waitB {st.mean(r[7] for r in rows):.0f} waitT {st.mean(r[8] for r in rows):.0f} busy {st.mean(busy):.0f}")
PY
