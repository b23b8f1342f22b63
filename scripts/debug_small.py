"""Minimal forward for debugging under compute-sanitizer: python scripts/debug_small.py [N h d_ff E]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import workload as W
from paper_2503_08467_b200 import MoEShardLayer

N, h, d_ff, E = (int(a) for a in (sys.argv[1:5] if len(sys.argv) > 4 else (1000, 256, 512, 8)))
torch.cuda.set_device(0)
inp = W.make_layer_inputs(11, N, h, d_ff, E, dtype=torch.bfloat16, device="cuda", routing="uniform")
L = MoEShardLayer(h, d_ff, E, max_tokens_per_rank=N, dtype=torch.bfloat16)
L.load_expert_shards(0, inp.w_i, inp.w_o)
y = L.forward(0, inp.x, inp.w_r, forced_expert=inp.forced)
torch.cuda.synchronize()
print("ok", y.float().abs().mean().item())
