"""Kernel timeline of pipelined forwards (torch profiler / CUPTI timestamps), bench c2 shapes,
3 rotating weight sets (> L2 between reuses)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
import workload as W
from paper_2503_08467_b200 import MoEShardLayer
import argparse
ap = argparse.ArgumentParser()
ap.add_argument("--E", type=int, default=64); ap.add_argument("--h", type=int, default=768)
ap.add_argument("--dff", type=int, default=3072); ap.add_argument("--N", type=int, default=8192)
ap.add_argument("--routing", default="natural"); ap.add_argument("--k", type=int, default=1)
a = ap.parse_args()
E, h, d_ff, N, NW = a.E, a.h, a.dff, a.N, 3
L = MoEShardLayer(h, d_ff, E, n_layers=NW, max_tokens_per_rank=N)
for l in range(NW):
    wi, wo = W.make_expert_weights(2, E, h, d_ff, device="cuda", layer=l); L.load_expert_shards(l, wi, wo); del wi, wo
x = W.make_tokens(2, N, h, device="cuda"); w_r = W.make_router_weight(2, h, E, device="cuda")
out = torch.empty_like(x)
forced = None if a.routing == "natural" else W.draw_experts(2, N, E, a.routing, device="cuda",
                                                            **({"k": a.k} if a.routing == "patho" else {}))
for k in range(30): L.forward(k % NW, x, w_r, forced_expert=forced, out=out)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as p:
    for k in range(12): L.forward(k % NW, x, w_r, forced_expert=forced, out=out)
    torch.cuda.synchronize()
p.export_chrome_trace("/tmp/trace.json")
ev = [e for e in json.load(open("/tmp/trace.json"))["traceEvents"] if e.get("cat") == "kernel"]
ev.sort(key=lambda e: e["ts"])
t0 = ev[0]["ts"]
for e in ev[:12]:
    print(f'{e["ts"]-t0:9.2f} {e["ts"]+e["dur"]-t0:9.2f} {e["dur"]:8.2f}  {e["name"][:60]}')
# per-kernel mean durations and step period
from collections import defaultdict
d = defaultdict(list)
for e in ev: d[e["name"][:40]].append(e["dur"])
for k, v in d.items(): print(f"{k:42s} n={len(v):3d} mean {sum(v)/len(v):8.2f} us")
starts = [e["ts"] for e in ev if "router" in e["name"]]
print("step period us:", [round(b - a, 1) for a, b in zip(starts, starts[1:])])
