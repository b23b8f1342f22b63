"""Per-step timeline of the e2e streaming loop (HostStreamer's schedule with timing events at
every boundary): H2D, forward and D2H start/end of a few steady-state steps, in us from the
first recorded step. Measurement only."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workload as W  # noqa: E402
from paper_2503_08467_b200 import MoEShardLayer  # noqa: E402

E, h, d_ff, N, SEED, STEPS, NB = 64, 768, 3072, 8192, 2, 60, 3


def main():
    dev = "cuda"
    layer = MoEShardLayer(h, d_ff, E, n_layers=1, max_tokens_per_rank=N, dtype=torch.bfloat16)
    wi, wo = W.make_expert_weights(SEED, E, h, d_ff, cols=(0, d_ff), device=dev, layer=0)
    layer.load_expert_shards(0, wi, wo)
    x = W.make_tokens(SEED, N, h, device=dev)
    w_r = W.make_router_weight(SEED, h, E, device=dev)
    xh = [x.cpu().pin_memory() for _ in range(2)]
    yh = [torch.empty_like(xh[0]).pin_memory() for _ in range(2)]
    din = [torch.empty_like(x) for _ in range(NB)]
    dout = [torch.empty_like(x) for _ in range(NB)]
    h2d, d2h = torch.cuda.Stream(), torch.cuda.Stream()
    comp = torch.cuda.current_stream()
    ev = lambda: torch.cuda.Event(enable_timing=True)
    T = [[ev() for _ in range(6)] for _ in range(STEPS)]
    fwd_done = [None] * STEPS
    out_free = [None] * STEPS
    import time
    host = {"h2d": 0.0, "fwd": 0.0, "d2h": 0.0}
    for k in range(STEPS):
        b = k % NB
        c0 = time.perf_counter()
        t = T[k]
        if k >= NB:
            h2d.wait_event(fwd_done[k - NB])
        with torch.cuda.stream(h2d):
            t[0].record(h2d)
            din[b].copy_(xh[k % 2], non_blocking=True)
            t[1].record(h2d)
        c1 = time.perf_counter()
        comp.wait_event(t[1])
        if k >= NB:
            comp.wait_event(out_free[k - NB])
        t[2].record(comp)
        layer.forward(0, din[b], w_r, out=dout[b])
        t[3].record(comp)
        fwd_done[k] = t[3]
        c2 = time.perf_counter()
        d2h.wait_event(t[3])
        with torch.cuda.stream(d2h):
            t[4].record(d2h)
            yh[k % 2].copy_(dout[b], non_blocking=True)
            t[5].record(d2h)
        out_free[k] = t[5]
        c3 = time.perf_counter()
        if k >= 20:
            for n, d in (("h2d", c1 - c0), ("fwd", c2 - c1), ("d2h", c3 - c2)):
                host[n] += d * 1e6 / (STEPS - 20)
    torch.cuda.synchronize()
    print(json.dumps({"host_us_per_step": {n: round(v, 1) for n, v in host.items()}}))
    base = T[40][0]
    for k in range(40, 46):
        print(json.dumps({"step": k, **{n: round(base.elapsed_time(T[k][i]) * 1e3, 1) for i, n in
                          enumerate(["h2d_s", "h2d_e", "fwd_s", "fwd_e", "d2h_s", "d2h_e"])}}))
    print(json.dumps({"period_us": round(T[40][0].elapsed_time(T[59][0]) * 1e3 / 19, 1)}))
    layer.close()


if __name__ == "__main__":
    main()
