"""Kernel timeline of a few pipelined forwards (torch profiler / CUPTI timestamps)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
import workload as W
from paper_2503_08467_b200 import MoEShardLayer
E, h, d_ff, N = 64, 768, 3072, 8192
L = MoEShardLayer(h, d_ff, E, max_tokens_per_rank=N)
wi, wo = W.make_expert_weights(2, E, h, d_ff, device="cuda"); L.load_expert_shards(0, wi, wo); del wi, wo
x = W.make_tokens(2, N, h, device="cuda"); w_r = W.make_router_weight(2, h, E, device="cuda")
out = torch.empty_like(x)
for _ in range(5): L.forward(0, x, w_r, out=out)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as p:
    for _ in range(6): L.forward(0, x, w_r, out=out)
    torch.cuda.synchronize()
p.export_chrome_trace("/tmp/trace.json")
ev = [e for e in json.load(open("/tmp/trace.json"))["traceEvents"] if e.get("cat") == "kernel"]
ev.sort(key=lambda e: e["ts"])
t0 = ev[0]["ts"]
for e in ev[:20]:
    print(f'{e["ts"]-t0:9.2f} {e["ts"]+e["dur"]-t0:9.2f} {e["dur"]:8.2f}  {e["name"][:60]}')
