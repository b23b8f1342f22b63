"""Per-kernel timeline of one MoE-layer forward (CUDA-graph replay, weights past L2) from
the -DMOESHARD_TIMELINE build (scripts/build_variant.sh tl -DMOESHARD_TIMELINE): globaltimer
stamps of kernel milestones, earliest / latest over CTAs, relative to the router's first CTA.
usage: python scripts/timeline_probe.py <shape> [routing]  (shapes of scripts/probe_multi.py)"""
import ctypes, json, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workload as W
from paper_2503_08467_b200 import MoEShardLayer, shard_columns
from paper_2503_08467_b200 import moeshard as C
from probe_multi import SHAPES

name = sys.argv[1] if len(sys.argv) > 1 else "c2g1"
routing = sys.argv[2] if len(sys.argv) > 2 else "natural"
E, h, d_ff, N, G = SHAPES[name]
F = d_ff // G
NW = max(2, math.ceil(3 * 126 * 2**20 / (2 * E * h * F * 2)))
L = MoEShardLayer(h, F, E, n_layers=NW, max_tokens_per_rank=N, dtype=torch.bfloat16)
c0, c1 = shard_columns(d_ff, G, 0)
for j in range(NW):
    wi, wo = W.make_expert_weights(2, E, h, d_ff, cols=(c0, c1), device="cuda", layer=j % 3)
    L.load_expert_shards(j, wi, wo)
    del wi, wo
x = W.make_tokens(2, N, h, device="cuda")
w_r = W.make_router_weight(2, h, E, device="cuda")
out = torch.empty_like(x)
f = None if routing == "natural" else W.draw_experts(2, N, E, routing, device="cuda")
lib = ctypes.CDLL(C.LIB_PATH)
tls = {k: getattr(lib, "moeshard_tl_" + k) for k in ("router", "group", "ffn")}
graphs = []
for j in range(NW):
    L.forward(j, x, w_r, forced_expert=f, out=out)
torch.cuda.synchronize()
for j in range(NW):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        L.forward(j, x, w_r, forced_expert=f, out=out)
    graphs.append(g)
for g in graphs:
    g.replay()
torch.cuda.synchronize()
names = {"router": ["start/end", "after griddep_wait", "mainloop done"],
         "group": ["scan after wait", "grouping start/end", "tables published", "grp after wait", "grp before tables", "grp after tables", "grp ranks done"],
         "ffn": ["start/end", "tables read", "token producer go", "last MMA issued"]}
acc = {}
reps = 12
for r in range(reps):
    buf = {k: (ctypes.c_ulonglong * 16)() for k in tls}
    for k in tls:
        tls[k](None, 1)
    graphs[r % NW].replay()
    torch.cuda.synchronize()
    for k in tls:
        tls[k](buf[k], 0)
    t0 = buf["router"][0]
    for k, labels in names.items():
        for i, lab in enumerate(labels):
            lo, hi = buf[k][2 * i], buf[k][2 * i + 1]
            key = f"{k}: {lab}"
            a = acc.setdefault(key, [0.0, 0.0])
            a[0] += ((lo - t0) / 1e3 if lo != 2**64 - 1 else float("nan")) / reps
            a[1] += ((hi - t0) / 1e3 if hi else float("nan")) / reps
print(json.dumps({"shape": name, "routing": routing,
                  "us_from_router_start": {k: [round(v[0], 2), round(v[1], 2)] for k, v in acc.items()}}))
