"""Step 1 alone (the ROUTE stage of a world-1 layer: tcgen05 router + histograms), CUDA-graph
replay, µs per call, for the token counts one rank routes at G = 1..8 (C2 / C3 shapes).
usage: python scripts/router_probe.py"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workload as W
from paper_2503_08467_b200 import MoEShardLayer
from paper_2503_08467_b200 import moeshard as C


def time_route(E, h, n, reps=200):
    L = MoEShardLayer(h, 256, E, max_tokens_per_rank=n, dtype=torch.bfloat16)
    L.load_expert_shards(0, torch.zeros(E, h, 256, dtype=torch.bfloat16, device="cuda"),
                         torch.zeros(E, 256, h, dtype=torch.bfloat16, device="cuda"))
    x = W.make_tokens(3, n, h, device="cuda")
    w_r = W.make_router_weight(3, h, E, device="cuda")
    out = torch.empty_like(x)
    fwd = lambda: L.forward(0, x, w_r, out=out, stages=C.MOESHARD_STAGE_ROUTE)
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        for _ in range(3):
            fwd()
    torch.cuda.current_stream().wait_stream(st)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(10):
            fwd()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps // 10):
        g.replay()
    e.record()
    torch.cuda.synchronize()
    L.check()
    L.close()
    return round(s.elapsed_time(e) / reps * 1e3, 2)


res = {}
for name, E, h in (("c2", 64, 768), ("c3", 128, 768), ("c5", 128, 1024)):
    for n in (1024, 2048, 4096, 8192, 16384, 32768):
        res[f"{name}_n{n}"] = time_route(E, h, n)
print(json.dumps(res))
