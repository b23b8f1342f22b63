"""MOESHARD_FLAG_P2P across PROCESSES: two ranks in two processes on this one GPU, the
exchange regions mapped into each other's address space through CUDA IPC
(moeshard_p2p_export / _open / _connect via MoEShardLayer.p2p_connect_group over a gloo
process group), whole forwards run concurrently (dynamic FFN scheduling, since the two
processes' kernels share the GPU). The concatenated outputs must match the unsharded
oracle - the multi-process code path of a multi-GPU run, minus NVLink."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


G, N, H, DFF, E = 2, 1024, 256, 512, 16
SEEDS = (51, 52, 53)


def _worker(rank, port, q):
    try:
        import torch.distributed as dist
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=G)
        torch.cuda.set_device(0)
        import workload as W
        from paper_2503_08467_b200 import MoEShardLayer, shard_columns
        from paper_2503_08467_b200 import moeshard as C
        n = N // G
        L = MoEShardLayer(H, DFF, E, max_tokens_per_rank=n, dtype=torch.bfloat16, rank=rank,
                          world=G, device=0,
                          flags=C.MOESHARD_FLAG_P2P | C.MOESHARD_FLAG_DYNAMIC_SCHED)
        base = W.make_layer_inputs(SEEDS[0], N, H, DFF, E, dtype=torch.bfloat16, routing="zipf")
        c0, c1 = shard_columns(DFF, G, rank)
        L.load_expert_shards(0, base.w_i[:, :, c0:c1].cuda(), base.w_o[:, c0:c1, :].cuda())
        w_r = base.w_r.cuda()
        outs = []
        for seed in SEEDS:
            x = W.make_tokens(seed, N, H)[rank * n:(rank + 1) * n].cuda().contiguous()
            f = W.draw_experts(seed, N, E, "zipf")[rank * n:(rank + 1) * n].cuda().contiguous()
            dist.barrier()
            y = L.forward(0, x, w_r, forced_expert=f)
            L.check()
            outs.append(y.float().cpu().numpy())
        dist.barrier()
        L.close()
        q.put((rank, outs, None))
    except Exception as e:  # report, do not hang the parent
        import traceback
        q.put((rank, None, traceback.format_exc()))


def test_p2p_two_processes_ipc_match_oracle():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import oracle as O
    import workload as W
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(G)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(G):
        rank, outs, err = q.get(timeout=300)
        assert err is None, f"rank {rank}:\n{err}"
        res[rank] = outs
    for p in procs:
        p.join(timeout=60)
    base = W.make_layer_inputs(SEEDS[0], N, H, DFF, E, dtype=torch.bfloat16, routing="zipf")
    for i, seed in enumerate(SEEDS):
        x = W.make_tokens(seed, N, H)
        f = W.draw_experts(seed, N, E, "zipf")
        y_ref = O.moe_layer(x, base.w_r, base.w_i, base.w_o, forced=f.numpy())
        y = np.concatenate([res[r][i] for r in range(G)])
        err = O.max_abs_rel(y, y_ref)
        assert err <= 2e-2, f"seed {seed}: max-abs-rel {err:.3e}"
