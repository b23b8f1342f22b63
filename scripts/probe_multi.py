"""Same-box A/B helper: time several MoE-layer shapes on one GPU (world-1 layer of width
d_ff/G = what one rank of a G-GPU layer computes after the AllGather), CUDA-graph replay
over weight sets rotated past L2, forced uniform and Zipf(1.2) routing. One JSON line.
usage: python scripts/probe_multi.py [shape ...]   shapes: c2g1 c2g8 c3g4 c5g1 c5g8 c4g8"""
import json, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workload as W
from paper_2503_08467_b200 import MoEShardLayer, shard_columns

SHAPES = {"c2g1": (64, 768, 3072, 8192, 1), "c2g8": (64, 768, 3072, 8192, 8),
          "c3g4": (128, 768, 3072, 16384, 4), "c5g1": (128, 1024, 4096, 32768, 1),
          "c5g8": (128, 1024, 4096, 32768, 8), "c5g2": (128, 1024, 4096, 32768, 2),
          "c5g4": (128, 1024, 4096, 32768, 4), "c4g8": (256, 768, 3072, 16384, 8),
          "c3g1": (128, 768, 3072, 16384, 1), "c3g8": (128, 768, 3072, 16384, 8),
          "c2r1k": (64, 768, 3072, 1024, 8)}   # one G = 8 rank's own 1024 tokens (router timeline)
# "<shape>k2": the same layer with top-2 routing (R21), natural router only


def probe(E, h, d_ff, N, G, steps=120, top_k=1):
    F = d_ff // G
    NW = max(1, math.ceil(3 * 126 * 2**20 / (2 * E * h * F * 2)))
    L = MoEShardLayer(h, F, E, n_layers=NW, max_tokens_per_rank=N, dtype=torch.bfloat16,
                      flags=int(os.environ.get("PROBE_FLAGS", "0")),
                      top_k=top_k)
    c0, c1 = shard_columns(d_ff, G, 0)
    for j in range(NW):
        wi, wo = W.make_expert_weights(2, E, h, d_ff, cols=(c0, c1), device="cuda", layer=j % 3)
        L.load_expert_shards(j, wi, wo)
        del wi, wo
    x = W.make_tokens(2, N, h, device="cuda")
    w_r = W.make_router_weight(2, h, E, device="cuda")
    out = torch.empty_like(x)
    res = {}
    for routing in (("uniform", "zipf") if top_k == 1 else ("natural",)):
        f = W.draw_experts(2, N, E, routing, device="cuda") if routing != "natural" else None
        fwd = lambda k: L.forward(k % NW, x, w_r, forced_expert=f, out=out)
        st = torch.cuda.Stream()
        st.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(st):
            for k in range(NW + 3):
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
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(reps):
            g.replay()
        e.record()
        torch.cuda.synchronize()
        res[routing] = round(s.elapsed_time(e) / (reps * NW) * 1e3, 2)
    L.check()
    L.close()
    return res


if __name__ == "__main__":
    names = sys.argv[1:] or ["c2g1", "c2g8", "c5g1"]
    print(json.dumps({n: probe(*SHAPES[n.replace("k2", "")], top_k=2 if n.endswith("k2") else 1)
                      for n in names}), flush=True)
