"""Kernel timeline of pipelined forwards (torch profiler / CUPTI timestamps), bench c2 shapes,
3 rotating weight sets (> L2 between reuses)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
import workload as W
from paper_2503_08467_b200 import MoEShardLayer
E, h, d_ff, N, NW = 64, 768, 3072, 8192, 3
L = MoEShardLayer(h, d_ff, E, n_layers=NW, max_tokens_per_rank=N)
for l in range(NW):
    wi, wo = W.make_expert_weights(2, E, h, d_ff, device="cuda", layer=l); L.load_expert_shards(l, wi, wo); del wi, wo
x = W.make_tokens(2, N, h, device="cuda"); w_r = W.make_router_weight(2, h, E, device="cuda")
out = torch.empty_like(x)
for k in range(30): L.forward(k % NW, x, w_r, out=out)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as p:
    for k in range(12): L.forward(k % NW, x, w_r, out=out)
    torch.cuda.synchronize()
p.export_chrome_trace("/tmp/trace.json")
ev = [e for e in json.load(open("/tmp/trace.json"))["traceEvents"] if e.get("cat") == "kernel"]
ev.sort(key=lambda e: e["ts"])
t0 = ev[0]["ts"]
for e in ev[:24]:
    print(f'{e["ts"]-t0:9.2f} {e["ts"]+e["dur"]-t0:9.2f} {e["dur"]:8.2f}  {e["name"][:60]}')
# per-kernel mean durations and step period
from collections import defaultdict
d = defaultdict(list)
for e in ev: d[e["name"][:40]].append(e["dur"])
for k, v in d.items(): print(f"{k:42s} n={len(v):3d} mean {sum(v)/len(v):8.2f} us")
starts = [e["ts"] for e in ev if "router" in e["name"]]
print("step period us:", [round(b - a, 1) for a, b in zip(starts, starts[1:])])
