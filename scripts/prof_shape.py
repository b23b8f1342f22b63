"""Run one world-1 layer shape a few times (for ncu captures of a single kernel).
usage: python scripts/prof_shape.py N h F E [flags] [routing]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workload as W
from paper_2503_08467_b200 import MoEShardLayer

N, h, F, E = (int(v) for v in sys.argv[1:5])
flags = int(sys.argv[5], 0) if len(sys.argv) > 5 else 0
routing = sys.argv[6] if len(sys.argv) > 6 else "uniform"
L = MoEShardLayer(h, F, E, n_layers=3, max_tokens_per_rank=N, dtype=torch.bfloat16, flags=flags)
for j in range(3):
    wi, wo = W.make_expert_weights(2, E, h, F, device="cuda", layer=j)
    L.load_expert_shards(j, wi, wo)
x = W.make_tokens(2, N, h, device="cuda")
w_r = W.make_router_weight(2, h, E, device="cuda")
f = W.draw_experts(2, N, E, routing, device="cuda")
for k in range(12):
    L.forward(k % 3, x, w_r, forced_expert=f)
torch.cuda.synchronize()
print("ok")
