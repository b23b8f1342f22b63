"""Time one MoE-layer shape on one GPU (a world=1 layer; with --G the d_ff/G shard a
rank computes after the AllGather): step time over rotating weight sets (>= 3x L2,
so weights stream from HBM), phase breakdown, routing in {uniform, zipf}.
usage: python scripts/shape_probe.py E h d_ff N [G] [steps]"""
import json, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workload as W
from paper_2503_08467_b200 import MoEShardLayer, shard_columns

E, h, d_ff, N = (int(a) for a in sys.argv[1:5])
G = int(sys.argv[5]) if len(sys.argv) > 5 else 1
steps = int(sys.argv[6]) if len(sys.argv) > 6 else 200
F = d_ff // G
wbytes = 2 * E * h * F * 2
NW = max(1, math.ceil(3 * 126 * 2**20 / wbytes))
seed = 2
L = MoEShardLayer(h, F, E, n_layers=NW, max_tokens_per_rank=N, dtype=torch.bfloat16)
c0, c1 = shard_columns(d_ff, G, 0)
for j in range(NW):
    wi, wo = W.make_expert_weights(seed, E, h, d_ff, cols=(c0, c1), device="cuda", layer=j % 3)
    L.load_expert_shards(j, wi, wo)
    del wi, wo
x = W.make_tokens(seed, N, h, device="cuda")
w_r = W.make_router_weight(seed, h, E, device="cuda")
out = torch.empty_like(x)
res = {"E": E, "h": h, "d_ff": d_ff, "N": N, "G": G, "F": F, "weight_sets": NW,
       }
for routing in ("uniform", "zipf"):
    f = W.draw_experts(seed, N, E, routing, device="cuda")
    fwd = lambda k: L.forward(k % NW, x, w_r, forced_expert=f, out=out)
    for k in range(20):
        fwd(k)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for k in range(steps):
        fwd(k)
    e.record()
    torch.cuda.synchronize()
    us = s.elapsed_time(e) / steps * 1e3
    # CUDA-graph replay of NW forwards (one per weight set), as bench.py times it
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        for k in range(NW):
            fwd(k)
    torch.cuda.current_stream().wait_stream(st)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for k in range(NW):
            fwd(k)
    reps = max(1, steps // NW)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        g.replay()
    e.record()
    torch.cuda.synchronize()
    us_graph = s.elapsed_time(e) / (reps * NW) * 1e3
    L.profile(True)
    for k in range(min(steps, 500)):
        fwd(k)
    ph, cnt = L.phase_ms()
    L.profile(False)
    res[routing] = {"step_us": round(us_graph, 2), "step_us_eager": round(us, 2),
                    "phases_us": {k: round(1e3 * v / max(cnt, 1), 2) for k, v in ph.items()},
                    "stats": L.stats()}
print(json.dumps(res))
