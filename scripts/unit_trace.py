"""Per-unit trace of the fused FFN (-DMOESHARD_TIMELINE build): for every cluster's first
16 units, the MMA warp's and the epilogue's globaltimer stamps, summarised per unit type.
usage: python scripts/unit_trace.py <shape> [routing]"""
import ctypes, json, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import workload as W
from paper_2503_08467_b200 import MoEShardLayer, shard_columns
from paper_2503_08467_b200 import moeshard as C
from probe_multi import SHAPES

name = sys.argv[1] if len(sys.argv) > 1 else "c2g8"
routing = sys.argv[2] if len(sys.argv) > 2 else "natural"
E, h, d_ff, N, G = SHAPES[name]
F = d_ff // G
NW = max(2, math.ceil(3 * 126 * 2**20 / (2 * E * h * F * 2)))
L = MoEShardLayer(h, F, E, n_layers=NW, max_tokens_per_rank=N, dtype=torch.bfloat16)
c0, c1 = shard_columns(d_ff, G, 0)
for j in range(NW):
    wi, wo = W.make_expert_weights(2, E, h, d_ff, cols=(c0, c1), device="cuda", layer=j % 3)
    L.load_expert_shards(j, wi, wo)
x = W.make_tokens(2, N, h, device="cuda")
w_r = W.make_router_weight(2, h, E, device="cuda")
out = torch.empty_like(x)
f = None if routing == "natural" else W.draw_experts(2, N, E, routing, device="cuda")
lib = ctypes.CDLL(C.LIB_PATH)
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
tl = (ctypes.c_ulonglong * 16)()
tr = (ctypes.c_ulonglong * (148 * 16 * 8))()
lib.moeshard_tl_ffn(None, 1)
lib.moeshard_tr_ffn(None, 1)
graphs[1 % NW].replay()
torch.cuda.synchronize()
lib.moeshard_tl_ffn(tl, 0)
lib.moeshard_tr_ffn(tr, 0)
t0 = tl[0]
a = np.array(tr, dtype=np.float64).reshape(148, 16, 8)
valid = a[:, :, 0] > 0
a = np.where(a > 0, (a - t0) / 1e3, np.nan)
st = L.stats()
n_mp_up = (F // 128 + 1) // 2
r = L.routing(N)
chunks = None
res = {"shape": name, "routing": routing, "ffn_us": (tl[1] - tl[0]) / 1e3,
       "tables_read_us": [(tl[2] - t0) / 1e3, (tl[3] - t0) / 1e3]}
ncl = 74
# unit index of slot k of cluster c = c + k * ncl (static schedule); up units first
total_up = st["tiles_up"] // (2 * n_mp_up) * n_mp_up if False else None
rows = []
for c in range(ncl):
    for k in range(16):
        if not valid[c, k]:
            continue
        t = a[c, k]
        rows.append(dict(c=c, k=k, u=c + k * ncl, tempty_wait=t[1] - t[0], b_wait=t[2] - t[1],
                         a_wait=t[3] - t[2], mma=t[4] - t[3], epi_lag=t[5] - t[4], epi=t[6] - t[5],
                         start=t[0], end_mma=t[4], h_ready=t[7]))
import collections
agg = collections.defaultdict(list)
for rr in rows:
    for kk in ("tempty_wait", "b_wait", "a_wait", "mma", "epi_lag", "epi"):
        agg[(rr["k"], kk)].append(rr[kk])
res["per_slot_mean_us"] = {f"k{k}": {kk: round(float(np.nanmean(agg[(k, kk)])), 2)
                                      for kk in ("tempty_wait", "b_wait", "a_wait", "mma", "epi_lag", "epi")}
                           for k in range(16) if (k, "mma") in agg}
ends = [max((rr["end_mma"] for rr in rows if rr["c"] == c), default=0) for c in range(ncl)]
res["cluster_last_mma_us"] = {"min": round(min(ends), 2), "max": round(max(ends), 2),
                              "mean": round(float(np.mean(ends)), 2)}
res["first_unit_start_us"] = round(float(np.nanmin(a[:, 0, 0])), 2)
res["first_mma_us"] = {"min": round(float(np.nanmin(a[:, 0, 3])), 2), "max": round(float(np.nanmax(a[:, 0, 3])), 2)}
print(json.dumps(res))
