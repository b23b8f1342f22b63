"""Where the e2e leg of bench.py loses time against the PCIe floor (scripts/pcie_bw.py): the c2
layer streamed from pinned host memory through MoEShardLayer.host_streamer with NBUF device
buffers, against the same copies with no forward and the forward with no copies. Measurement
only; prints one JSON line per case."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workload as W  # noqa: E402
from paper_2503_08467_b200 import MoEShardLayer  # noqa: E402

E, h, d_ff, N, SEED, STEPS = 64, 768, 3072, 8192, 2, 200


def timed(fn, finish):
    for k in range(10):
        fn(k)
    finish()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for k in range(STEPS):
        fn(k)
    finish()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / STEPS


def main():
    dev = "cuda"
    layer = MoEShardLayer(h, d_ff, E, n_layers=1, max_tokens_per_rank=N, dtype=torch.bfloat16)
    wi, wo = W.make_expert_weights(SEED, E, h, d_ff, cols=(0, d_ff), device=dev, layer=0)
    layer.load_expert_shards(0, wi, wo)
    x = W.make_tokens(SEED, N, h, device=dev)
    w_r = W.make_router_weight(SEED, h, E, device=dev)
    out = torch.empty_like(x)
    xh = [x.cpu().pin_memory() for _ in range(2)]
    yh = [torch.empty_like(xh[0]).pin_memory() for _ in range(2)]
    res = {}
    res["forward_only"] = timed(lambda k: layer.forward(0, x, w_r, out=out), lambda: None)
    st = layer.host_streamer(N)
    res["host_streamer"] = timed(lambda k: st.step(0, xh[k % 2], w_r, yh[k % 2]), st.join)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    cur = torch.cuda.current_stream()

    def copies(k):
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            x.copy_(xh[k % 2], non_blocking=True)
        with torch.cuda.stream(s2):
            yh[k % 2].copy_(out, non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)
    res["copies_only"] = timed(copies, lambda: None)
    x2, o2 = x.clone(), out.clone()

    def overlapped(k):   # the same copies on other buffers, with an independent forward
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            x2.copy_(xh[k % 2], non_blocking=True)
        with torch.cuda.stream(s2):
            yh[k % 2].copy_(o2, non_blocking=True)
        layer.forward(0, x, w_r, out=out)
        cur.wait_stream(s1)
        cur.wait_stream(s2)
    res["copies_with_independent_forward"] = timed(overlapped, lambda: None)
    # lock-step software pipeline: step k issues H2D(k+1), D2H(k-1) and forward(k) together,
    # and the next step waits for all three (period = max(copies in both directions, forward))
    din = [torch.empty_like(x) for _ in range(3)]
    dout = [torch.empty_like(x) for _ in range(3)]

    def lockstep(k):
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            din[(k + 1) % 3].copy_(xh[(k + 1) % 2], non_blocking=True)
        with torch.cuda.stream(s2):
            yh[(k - 1) % 2].copy_(dout[(k - 1) % 3], non_blocking=True)
        layer.forward(0, din[k % 3], w_r, out=dout[k % 3])
        cur.wait_stream(s1)
        cur.wait_stream(s2)
    res["lockstep_pipeline"] = timed(lockstep, lambda: None)
    for k, v in res.items():
        print(json.dumps({"case": k, "us_per_step": round(v, 1), "tokens_per_s": round(N / (v * 1e-6))}))
    layer.close()


if __name__ == "__main__":
    main()
