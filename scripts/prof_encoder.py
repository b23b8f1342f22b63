import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
import workload as W
from harness.encoder import EncoderConfig, SwitchEncoder
from paper_2503_08467_b200 import MoEShardLayer
cfg = EncoderConfig()
fac = lambda m, n: MoEShardLayer(cfg.d_model, cfg.d_ff, cfg.n_experts, n_layers=m, max_tokens_per_rank=n)
enc = SwitchEncoder(cfg, seed=3, device="cuda", moe_layer_factory=fac)
x = W.make_tokens(3, cfg.batch * cfg.seq, cfg.d_model, device="cuda").view(cfg.batch, cfg.seq, cfg.d_model)
for _ in range(3): enc.forward(x)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as p:
    enc.forward(x); torch.cuda.synchronize()
print(p.key_averages().table(sort_by="cuda_time_total", row_limit=15, max_name_column_width=60))
