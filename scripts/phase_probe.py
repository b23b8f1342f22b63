"""Per-phase times (phase CUDA events of the library, eager forwards) of a world-1 layer with
the given flags - e.g. the exchange paths' own cost at G = 1 (MOESHARD_FLAG_P2P = 512,
FORCE_COLLECTIVES = 1). usage: python scripts/phase_probe.py <shape> <flags>"""
import json, math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workload as W
from paper_2503_08467_b200 import MoEShardLayer, shard_columns
from probe_multi import SHAPES

name = sys.argv[1] if len(sys.argv) > 1 else "c2g1"
flags = int(sys.argv[2]) if len(sys.argv) > 2 else 0
E, h, d_ff, N, G = SHAPES[name]
F = d_ff // G
NW = max(1, math.ceil(3 * 126 * 2**20 / (2 * E * h * F * 2)))
L = MoEShardLayer(h, F, E, n_layers=NW, max_tokens_per_rank=N, dtype=torch.bfloat16, flags=flags)
if flags & 512:
    MoEShardLayer.p2p_connect_local([L])
c0, c1 = shard_columns(d_ff, G, 0)
for j in range(NW):
    wi, wo = W.make_expert_weights(2, E, h, d_ff, cols=(c0, c1), device="cuda", layer=j % 3)
    L.load_expert_shards(j, wi, wo)
x = W.make_tokens(2, N, h, device="cuda")
w_r = W.make_router_weight(2, h, E, device="cuda")
f = W.draw_experts(2, N, E, "uniform", device="cuda")
out = torch.empty_like(x)
for k in range(10):
    L.forward(k % NW, x, w_r, forced_expert=f, out=out)
res = []
for rep in range(3):
    torch.cuda.synchronize()
    time.sleep(0.3)
    L.profile(True)
    for k in range(40):
        L.forward(k % NW, x, w_r, forced_expert=f, out=out)
    ph, cnt = L.phase_ms()
    L.profile(False)
    res.append({k: round(1e3 * v / max(cnt, 1), 2) for k, v in ph.items()})
L.check()
print(json.dumps({"shape": name, "flags": flags, "phases_us": res[1]}))
