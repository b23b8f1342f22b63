"""MoEShard vs the expert-parallel baseline (Fig. 1) and MoEShard with vs
without the Sec. 3.3 launch fusion (Fig. 2) on the paper's sweep:
Switch-Base shapes (h=768, d_ff=3072), seq 120, the paper's skewed router (alpha_r = 0.6,
k_r = 10% of E), E = 8..256 at batch 250 and batch 10..450 at E = 128,
|G| = 4 GPUs as in the paper.

One B200 is available, so the G ranks are virtual: G contexts of the same transport (peer
memory) share the GPU and are driven stage by stage (ROUTE on every rank, then COMPUTE, then
REDUCE); every stage of every rank is timed alone with CUDA events, i.e. as if each rank had
the whole GPU. Per system and point:
  compute_us   max over ranks of the COMPUTE stage (grouping + grouped FFN) - where EP's
               imbalance shows (a hot host computes most tokens)
  route_us / reduce_us  max over ranks of the other two stages (router + push / dispatch;
               aggregate / combine - on one GPU the pushes are local copies)
  nvlink_us    the exchange at 900 GB/s per direction: per rank max(bytes sent, received) of
               Step 3 + Step 5 (MoEShard: (G-1) n h 2 B each way per collective; EP: the
               rows actually dispatched / returned, from the admission tables)
  layer_us     route + compute + reduce + nvlink (no overlap assumed for either system)
and the MoE-layer speedup EP / MoEShard. The ablation rows run MoEShard with one up + one
down launch per expert ("per_expert": the paper's "without MegaBlocks", 2E launches) and per
(source rank, expert) ("per_source": 2EG launches) instead of the one fused grouped launch;
their exchange is MoEShard's. TTFT differs from 6 x layer_us by the non-MoE
blocks, identical (replicated) in both systems. Dropped tokens (EP, E > 50) are reported.
usage: python scripts/ep_sweep.py [--quick] > profiles/r02/ep_sweep.json"""
import argparse, json, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import workload as W
from paper_2503_08467_b200 import MoEShardLayer, shard_columns
from paper_2503_08467_b200 import moeshard as C

H, DFF, SEQ, G = 768, 3072, 120, 4
NV_GBS = 900.0
L2 = 126 * 2**20


KINDS = {"moeshard": 0, "per_expert": C.MOESHARD_FLAG_LAUNCH_PER_EXPERT,
         "per_source": C.MOESHARD_FLAG_LAUNCH_PER_SOURCE, "ep": C.MOESHARD_FLAG_EXPERT_PARALLEL}


def make_system(kind, E, n, n_layers, seed):
    flags = C.MOESHARD_FLAG_P2P | KINDS[kind]
    layers = [MoEShardLayer(H, DFF, E, n_layers=n_layers, max_tokens_per_rank=n,
                            dtype=torch.bfloat16, rank=r, world=G, flags=flags) for r in range(G)]
    MoEShardLayer.p2p_connect_local(layers)
    El = E // G
    for j in range(n_layers):
        for r, L in enumerate(layers):
            if kind == "ep":
                wi, wo = W.make_expert_weights(seed + j, E, H, DFF, device="cuda",
                                               experts=range(r * El, (r + 1) * El))
            else:
                wi, wo = W.make_expert_weights(seed + j, E, H, DFF, cols=shard_columns(DFF, G, r),
                                               device="cuda")
            L.load_expert_shards(j, wi, wo)
            del wi, wo
    return layers


def run(layers, xs, fs, w_r, n_layers, reps=8, warmup=3):
    stages = (C.MOESHARD_STAGE_ROUTE, C.MOESHARD_STAGE_COMPUTE, C.MOESHARD_STAGE_REDUCE)
    ys = [torch.empty_like(x) for x in xs]
    acc = np.zeros((3, G))
    for it in range(warmup + reps):
        j = it % n_layers
        ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(G)] for _ in stages]
        for si, st in enumerate(stages):
            for r, L in enumerate(layers):
                ev[si][r][0].record()
                L.forward(j, xs[r], w_r, forced_expert=fs[r], out=ys[r], stages=st)
                ev[si][r][1].record()
        torch.cuda.synchronize()
        if it >= warmup:
            acc += np.array([[a.elapsed_time(b) * 1e3 for a, b in row] for row in ev])
    for L in layers:
        L.check()
    return acc / reps, ys


def point(E, batch, seed=7):
    N = batch * SEQ
    n = N // G
    N = n * G
    El = E // G
    k_r = max(1, round(0.1 * E))
    x = W.make_tokens(seed, N, H, device="cuda")
    w_r = W.make_router_weight(seed, H, E, device="cuda")
    f = W.draw_experts(seed, N, E, "skew", device="cuda", alpha_r=0.6, k_r=k_r)
    xs = [x[r * n:(r + 1) * n].contiguous() for r in range(G)]
    fs = [f[r * n:(r + 1) * n].contiguous() for r in range(G)]
    per_rank_w = 2 * E * H * (DFF // G) * 2
    NL = max(1, min(6, math.ceil(3 * L2 / per_rank_w)))
    res = {"E": E, "batch": batch, "seq": SEQ, "tokens": N, "G": G, "k_r": k_r, "alpha_r": 0.6,
           "weight_sets": NL}
    row_bytes = H * 2
    for kind in KINDS:
        layers = make_system(kind, E, n, NL, seed)
        t, ys = run(layers, xs, fs, w_r, NL)
        if kind != "ep":
            sent = recv = 2 * (G - 1) * n * row_bytes          # AG + RS, per rank, each direction
            drops, load = 0, [N] * G                           # every rank computes all N tokens
        else:
            adm = [L.ep_admission(n) for L in layers]
            owner = [a["owner"].cpu().numpy() for a in adm]
            load = [int(layers[o].ep_admission(n)["received"].sum()) for o in range(G)]
            drops = int(sum((ow < 0).sum() for ow in owner))
            # dispatch: rank r sends rows whose host o != r; host o receives them; combine mirrors it
            out_b = [int(((ow >= 0) & (ow != r)).sum()) * row_bytes for r, ow in enumerate(owner)]
            in_b = [sum(int((owner[r] == o).sum()) for r in range(G) if r != o) * row_bytes
                    for o in range(G)]
            sent = max(max(o + i for o, i in zip(out_b, in_b)), 0)   # per rank: step 3 out + step 5 in
            recv = sent
        nv = max(sent, recv) / (NV_GBS * 1e3)
        route, comp, red = (float(t[i].max()) for i in range(3))
        res[kind] = {"route_us": round(route, 2), "compute_us": round(comp, 2),
                     "compute_us_per_rank": [round(float(v), 2) for v in t[1]],
                     "reduce_us": round(red, 2), "nvlink_us": round(nv, 2),
                     "layer_us": round(route + comp + red + nv, 2),
                     "tokens_computed_per_rank": load, "dropped_tokens": drops}
        for L in layers:
            L.close()
        torch.cuda.synchronize()
    res["speedup_layer"] = round(res["ep"]["layer_us"] / res["moeshard"]["layer_us"], 3)
    res["speedup_compute"] = round(res["ep"]["compute_us"] / res["moeshard"]["compute_us"], 3)
    res["fusion_gain_per_expert"] = round(res["per_expert"]["layer_us"] / res["moeshard"]["layer_us"], 3)
    res["fusion_gain_per_source"] = round(res["per_source"]["layer_us"] / res["moeshard"]["layer_us"], 3)
    print(json.dumps({k: res[k] for k in ("E", "batch", "speedup_layer", "speedup_compute",
                                          "fusion_gain_per_expert", "fusion_gain_per_source")}),
          file=sys.stderr, flush=True)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    a = ap.parse_args()
    experts = [8, 32, 128] if a.quick else [8, 16, 32, 64, 128, 256]
    batches = [10, 250] if a.quick else [10, 50, 100, 200, 300, 450]
    torch.cuda.set_device(0)
    out = {"note": __doc__.split("usage")[0].strip(), "vary_experts": [point(E, 250) for E in experts],
           "vary_batch": [point(128, b) for b in batches]}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
