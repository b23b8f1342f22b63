"""Per-rank load-balance invariance on ONE GPU (SURVEY.md §8(d) C4 checks 2-4).

Rank g of a G-GPU MoEShard layer computes, after the AllGather, the Switch MoE
layer of ALL N tokens against its d_ff/G column shard. That
compute is a world=1 layer with d_ff/G and N tokens, so each virtual rank g is
timed here on its own weight shard: per-rank compute time max/min, tile counts
(exactly equal by construction) and skewed/uniform time ratios. Collectives are
not included (one GPU). Writes one JSON document to stdout.
"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workload as W
from paper_2503_08467_b200 import MoEShardLayer, shard_columns

CASES = {   # name: (E, h, d_ff, N, G, seed, routings)
    "c4_g8": (256, 768, 3072, 16384, 8, 4, ["uniform", ("patho", {"k": 1}), ("patho", {"k": 3}), "skew",
                                             ("zipf", {"s": 1.2})]),
    "c2_g8": (64, 768, 3072, 8192, 8, 2, ["uniform", ("zipf", {"s": 1.2})]),
    "c2_g4": (64, 768, 3072, 8192, 4, 2, ["uniform", ("zipf", {"s": 1.2})]),
    "c2_g2": (64, 768, 3072, 8192, 2, 2, ["uniform", ("zipf", {"s": 1.2})]),
    "c3_g8": (128, 768, 3072, 16384, 8, 3, ["uniform", ("zipf", {"s": 1.2}), "skew"]),
    "c5_g8": (128, 1024, 4096, 32768, 8, 5, ["uniform", ("zipf", {"s": 1.2})]),
}


def graph_of(L, x, w_r, forced, out, nw):
    """One CUDA graph holding nw forwards over the rotating weight sets (>= 3x L2 in total),
    so every forward streams its weights from HBM and launches cost nothing."""
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        for k in range(nw + 2):
            L.forward(k % nw, x, w_r, forced_expert=forced, out=out)
    torch.cuda.current_stream().wait_stream(st)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for k in range(nw):
            L.forward(k % nw, x, w_r, forced_expert=forced, out=out)
    return g


def time_graph(g, nw, reps):
    for _ in range(2):
        g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        g.replay()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / (reps * nw) * 1e3   # us per forward


def main():
    names = sys.argv[1:] or list(CASES)
    res = {}
    for name in names:
        E, h, d_ff, N, G, seed, routings = CASES[name]
        F = d_ff // G
        x = W.make_tokens(seed, N, h, device="cuda")
        w_r = W.make_router_weight(seed, h, E, device="cuda")
        out = torch.empty_like(x)
        layers = []
        nw = max(1, -(-3 * 126 * 2**20 // (2 * E * h * F * 2)))
        for g in range(G):
            c0, c1 = shard_columns(d_ff, G, g)
            L = MoEShardLayer(h, F, E, n_layers=nw, max_tokens_per_rank=N, dtype=torch.bfloat16)
            for j in range(nw):
                wi, wo = W.make_expert_weights(seed, E, h, d_ff, cols=(c0, c1), device="cuda", layer=j)
                L.load_expert_shards(j, wi, wo)
                del wi, wo
            layers.append(L)
        case = {"E": E, "h": h, "d_ff": d_ff, "N": N, "G": G, "d_ff_per_rank": F, "weight_sets": nw,
                "note": "each virtual rank = the world-1 layer of all N tokens on its d_ff/G shard "
                        "(what a rank computes after the AllGather); collectives not included; "
                        "CUDA-graph replay of weight_sets forwards, median of 5 interleaved rounds per rank",
                "routings": {}}
        for r in routings:
            rname, kw = (r, {}) if isinstance(r, str) else r
            forced = W.draw_experts(seed, N, E, rname, device="cuda", **kw)
            label = rname + "".join(f"_{k}{v}" for k, v in kw.items())
            graphs = [graph_of(L, x, w_r, forced, out, nw) for L in layers]
            reps = max(2, 60 // nw)
            samples = [[] for _ in layers]
            for _ in range(5):          # ranks interleaved, 5 rounds: clock / power drift cancels
                for gi, g in enumerate(graphs):
                    samples[gi].append(time_graph(g, nw, reps))
            t = [sorted(v)[len(v) // 2] for v in samples]
            tiles = []
            for L in layers:
                L.forward(0, x, w_r, forced_expert=forced, out=out)
                st = L.stats()
                tiles.append((st["tiles_up"], st["tiles_down"]))
            del graphs
            case["routings"][label] = {
                "rank_us": [round(v, 2) for v in t], "max_over_min": round(max(t) / min(t), 4),
                "tiles_equal_on_all_ranks": len(set(tiles)) == 1, "tiles": list(tiles[0]),
                "experts_active": int((torch.bincount(forced.long(), minlength=E) > 0).sum())}
        u = max(case["routings"]["uniform"]["rank_us"])
        for k, v in case["routings"].items():
            v["max_rank_time_over_uniform"] = round(max(v["rank_us"]) / u, 4)
        for L in layers:
            L.close()
        res[name] = case
        print(json.dumps({name: case}), file=sys.stderr, flush=True)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
