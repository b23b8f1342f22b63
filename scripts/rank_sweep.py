"""Per-rank compute time of a G-GPU MoEShard layer, measured on ONE GPU (CUDA-graph replay,
weights rotated past L2): what every rank computes - router on its n = N/G tokens, Step 2
and both grouped products over all N tokens on its d_ff/G shard. A world-1 layer of width
d_ff/G routes all N tokens it is given, so per rank = forward(N) - router(N) + router(n),
each term timed as its own graph (router alone = the ROUTE stage of a world-1 layer) -
for the BASELINE layer configs at G = 1, 2, 4, 8, uniform and Zipf(1.2) routing. The
exchange steps are NOT run (one GPU); the JSON adds the NVLink bytes per rank and their
time at the 770 GB/s measured peer bandwidth so a reader can bound the G > 1 layer time.
usage: python scripts/rank_sweep.py > profiles/r01_rank_sweep.json"""
import json, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workload as W
from paper_2503_08467_b200 import MoEShardLayer, shard_columns
from paper_2503_08467_b200 import moeshard as C

CFGS = {"c2": (64, 768, 3072, 8192), "c3": (128, 768, 3072, 16384), "c5": (128, 1024, 4096, 32768)}
PEER_GBS = 770.0


def per_rank(E, h, d_ff, N, G, steps=60):
    F = d_ff // G
    NW = max(1, math.ceil(3 * 126 * 2**20 / (2 * E * h * F * 2)))
    L = MoEShardLayer(h, F, E, n_layers=NW, max_tokens_per_rank=N, dtype=torch.bfloat16)
    c0, c1 = shard_columns(d_ff, G, 0)
    for j in range(NW):
        wi, wo = W.make_expert_weights(2, E, h, d_ff, cols=(c0, c1), device="cuda", layer=j % 3)
        L.load_expert_shards(j, wi, wo)
        del wi, wo
    x = W.make_tokens(2, N, h, device="cuda")
    w_r = W.make_router_weight(2, h, E, device="cuda")
    out = torch.empty_like(x)
    res = {}

    def graph_time(fn):
        st = torch.cuda.Stream()
        st.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(st):
            for k in range(NW + 3):
                fn(k)
        torch.cuda.current_stream().wait_stream(st)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for k in range(NW):
                fn(k)
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
        return s.elapsed_time(e) / (reps * NW) * 1e3

    n = N // G
    xn = x[:n].contiguous()
    route_N = graph_time(lambda k: L.forward(k % NW, x, w_r, out=out, stages=C.MOESHARD_STAGE_ROUTE))
    route_n = graph_time(lambda k: L.forward(k % NW, xn, w_r, out=out[:n], stages=C.MOESHARD_STAGE_ROUTE))
    res["router_us"] = {"N": round(route_N, 2), "n": round(route_n, 2)}
    for routing in ("uniform", "zipf"):
        f = W.draw_experts(2, N, E, routing, device="cuda")
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
        t_full = s.elapsed_time(e) / (reps * NW) * 1e3
        res[routing] = round(t_full - route_N + route_n, 2)
        res[routing + "_all_N_routed"] = round(t_full, 2)
    L.close()
    return res


def main():
    out = {"note": "per-rank compute only: forward(N) - router(N) + router(N/G) (graph replays; "
                   "*_all_N_routed keeps the router over all N); nvlink_us = (G-1)/G * N * h * 2 B * 2 (AllGather "
                   "+ ReduceScatter, bf16) / 770 GB/s", "configs": {}}
    for name, (E, h, d_ff, N) in CFGS.items():
        rows = {}
        for G in (1, 2, 4, 8):
            t = per_rank(E, h, d_ff, N, G)
            nv = (G - 1) / G * N * h * 2 * 2 / (PEER_GBS * 1e3)
            rows[G] = {"compute_us": t, "nvlink_us": round(nv, 2),
                       "tokens_per_s_compute_only": {r: round(N / t[r] * 1e6) for r in ("uniform", "zipf")}}
            print(name, G, rows[G], file=sys.stderr, flush=True)
        out["configs"][name] = {"E": E, "h": h, "d_ff": d_ff, "N": N, "by_G": rows}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
